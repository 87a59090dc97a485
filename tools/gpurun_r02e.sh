set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr_build.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > $O/r02e_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02e_gputest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02e_csr_launches.csv python tools/prof_csr.py --iters 2 > $O/r02e_csr.log 2>&1
tail -3 $O/r02e_gputest.log
