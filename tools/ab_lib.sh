# A/B of two in-tree builds on the same box: tools/ab_lib.sh [configs...]
CFGS=${@:-C5}
for lib in paper_2507_16991_b200/libgraphmill_b200.so paper_2507_16991_b200/libgraphmill_b200_varB.so; do
  echo "== $lib"
  for m in sum max; do GM_LIB_PATH=$PWD/$lib python tools/exp_heavy.py $m | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['ms'])"; done
  GM_LIB_PATH=$PWD/$lib python tools/bench_configs.py $CFGS 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d.get('reduce',''), round(d['ms'],3), round(d.get('frac_hbm',0),3))"
done
