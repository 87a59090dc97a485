# window cost 1024 (new default) vs 256: per-config SpMM lines (C2, C5, C3 relation; hashes must match) + full GPU suite + smoke
O=gpurun_out
R=r02win4
rm -f $O/${R}_ab.txt
for v in base w256; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; [ $v != base ] && lib=paper_2507_16991_b200/libgraphmill_b200_$v.so
  echo "$v $(GM_LIB_PATH=$PWD/$lib GM_AB_HASH=1 timeout 1500 python tools/bench_configs.py C3 C2 C2X C5 2>&1 | grep '"reduce"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['reduce'], round(d['ms'],3), d.get('out_hash'))" | tr '\n' ';')" >> $O/${R}_ab.txt
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${R}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${R}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O/${R}_gputest.log 2>&1
cat $O/${R}_ab.txt; tail -3 $O/${R}_gputest.log
