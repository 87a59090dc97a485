# dw slice kernel warps per CTA (GM_EDGE_DOT_WARPS 8 / 4 / 2), same box, hashes must match
O=gpurun_out
R=r02dww
rm -f $O/${R}_ab.txt
for rep in 1 2; do for w in 8 4 2; do
  echo "warps=$w $(GM_AB_DW_ONLY=1 GM_EDGE_DOT_WARPS=$w timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
