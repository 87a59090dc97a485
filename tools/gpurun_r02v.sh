O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist_push.py tests/test_gpu_dist_blocked.py tests/test_gpu_dist_nccl.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/r02v_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02v_gputest.log
python tools/ab_flat.py > $O/r02v_flat.json 2>&1
tail -25 $O/r02v_gputest.log; cat $O/r02v_flat.json
