O=gpurun_out
rm -f $O/r02c5b_ab.txt
timeout 900 python -m pytest tests/test_gpu_dist_push.py tests/test_gpu_dist_nccl.py -x -q -p no:cacheprovider > $O/r02c5b_test.log 2>&1; echo "pytest rc=$?" >> $O/r02c5b_test.log
for rep in 1 2; do for v in base noepi; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib timeout 600 python tools/bench_configs.py C5 C4 2>/dev/null | sed "s/^/$v /" >> $O/r02c5b_ab.txt
done; done
tail -2 $O/r02c5b_test.log; python -c "
import json
for l in open('$O/r02c5b_ab.txt'):
    v,j=l.split(' ',1); d=json.loads(j); print(v, d['config'][:10], d['reduce'], round(d['ms'],3))"
