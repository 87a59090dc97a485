# max sweep edges per batch (GM_FLAT_MAX_U 6 base / 5 / 7), max + argmax line, same box
O=gpurun_out
R=r02mu
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base mu5 mu7; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; [ $v != base ] && lib=paper_2507_16991_b200/libgraphmill_b200_$v.so
  GM_LIB_PATH=$PWD/$lib timeout 900 python bench.py --no-cpu-baseline  > $O/${R}_$v.json 2> $O/${R}_$v.err
  echo "$v $(python -c "import json;d=json.load(open('$O/${R}_$v.json'));print(d['ms_per_step'], d['secondary']['max_argmax_spmm']['ms'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
