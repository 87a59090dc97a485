# dw slice kernel entries per sub-batch (GM_DOT_SLICE_U 8 base / 6 / 10) with 2-warp CTAs, same box, hashes must match
O=gpurun_out
R=r02du
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base du6 du10; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; [ $v != base ] && lib=paper_2507_16991_b200/libgraphmill_b200_$v.so
  echo "$v $(GM_LIB_PATH=$PWD/$lib GM_AB_DW_ONLY=1 timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
