O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr_build.py tests/test_gpu_dist_build.py -x -q -p no:cacheprovider > $O/r02csr_test.log 2>&1; echo "pytest rc=$?" >> $O/r02csr_test.log
python tools/ab_csr.py > $O/r02csr_ab.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02csr_launch.csv python tools/prof_csr.py --iters 1 > /dev/null 2>&1
tail -1 $O/r02csr_test.log; cat $O/r02csr_ab.txt; grep rowptr $O/r02csr_launch.csv | awk -F'","' '{print $NF}'
