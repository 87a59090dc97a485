O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr_build.py -x -q -p no:cacheprovider > $O/r02f_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02f_gputest.log
GM_RADIX_BITS=8 timeout 900 python -m pytest tests/test_gpu_csr_build.py -x -q -p no:cacheprovider >> $O/r02f_gputest.log 2>&1; echo "pytest8 rc=$?" >> $O/r02f_gputest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02f_csr11.csv python tools/prof_csr.py --iters 1 > $O/r02f_csr.log 2>&1
GM_RADIX_BITS=8 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02f_csr8.csv python tools/prof_csr.py --iters 1 >> $O/r02f_csr.log 2>&1
python tools/ab_csr.py >> $O/r02f_csr.log 2>&1
GM_RADIX_BITS=8 python tools/ab_csr.py >> $O/r02f_csr.log 2>&1
tail -3 $O/r02f_gputest.log; tail -4 $O/r02f_csr.log
