# dw slice kernel entries per warp (GM_EDGE_DOT_PER_WARP) with 2-warp CTAs, same box, hashes must match
O=gpurun_out
R=r02pw
rm -f $O/${R}_ab.txt
for rep in 1 2; do for pw in 256 512 1024 128; do
  echo "per_warp=$pw $(GM_AB_DW_ONLY=1 GM_EDGE_DOT_PER_WARP=$pw timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
