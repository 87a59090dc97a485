set -x
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02u_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02u_gputest.log
timeout 900 python bench.py > $O/r02u_bench.json 2> $O/r02u_bench.err
tail -2 $O/r02u_gputest.log; tail -3 $O/r02u_bench.err
