set -x
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02o_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02o_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02o_smoke.log 2>&1
timeout 900 python bench.py > $O/r02o_bench.json 2> $O/r02o_bench.err
python tools/ab_backward.py > $O/r02o_bwd.json 2>&1
tail -2 $O/r02o_gputest.log; tail -1 $O/r02o_smoke.log
