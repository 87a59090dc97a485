O=gpurun_out
rm -f $O/r02dw4_ab.txt
for rep in 1 2; do for pw in 64 128 256 512 2048; do
  echo "pw=$pw $(GM_EDGE_DOT_SLICE=1 GM_EDGE_DOT_PER_WARP=$pw python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02dw4_ab.txt
done; done
cat $O/r02dw4_ab.txt
