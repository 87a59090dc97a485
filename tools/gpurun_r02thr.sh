# with 4-warp flat CTAs: hub threshold (GM_HEAVY_THR) and hub ring depth re-checked on the headline + max lines
O=gpurun_out
R=r02thr
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base thr512 thr2048 ring8; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; extra=""
  case $v in ring8) lib=paper_2507_16991_b200/libgraphmill_b200_$v.so;; thr512) extra="GM_HEAVY_THR=512";; thr2048) extra="GM_HEAVY_THR=2048";; esac
  env GM_LIB_PATH=$PWD/$lib $extra timeout 900 python bench.py --no-cpu-baseline > $O/${R}_$v.json 2> $O/${R}_$v.err
  echo "$v $(python -c "import json;d=json.load(open('$O/${R}_$v.json'));print(d['ms_per_step'], d['roofline']['frac'], d['secondary']['max_argmax_spmm']['ms'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
