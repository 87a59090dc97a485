# flat-kernel window cost (edges + rows per warp window: 256 base, 128, 512), sum and max lines
O=gpurun_out
R=r02win2
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base w512 w768 w1024; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so
  [ $v != base ] && lib=paper_2507_16991_b200/libgraphmill_b200_$v.so
  GM_LIB_PATH=$PWD/$lib timeout 900 python bench.py --no-cpu-baseline > $O/${R}_$v.json 2> $O/${R}_$v.err
  echo "$v $(python -c "import json;d=json.load(open('$O/${R}_$v.json'));print(d['ms_per_step'], d['secondary']['max_argmax_spmm']['ms'], d['secondary']['backward_max']['ms'], d['secondary']['backward_dw']['ms'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
