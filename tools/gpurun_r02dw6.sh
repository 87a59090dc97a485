# staged (cp.async ring) dw kernel: parity subset + same-box A/B against the slice kernel (bit hash compared)
O=gpurun_out
rm -f $O/r02dw6_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -p no:cacheprovider -k "backward or dw or weight or empty or slice" > $O/r02dw6_test.log 2>&1; echo "pytest rc=$?" >> $O/r02dw6_test.log
for rep in 1 2; do for cfg in 0 83 84 44 46 162 163; do
  echo "staged=$cfg $(GM_AB_DW_ONLY=1 GM_DOT_STAGED=$cfg timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02dw6_ab.txt
done; done
for cold in 0; do echo "staged=83 cold=$cold $(GM_AB_DW_ONLY=1 GM_DOT_STAGED_COLD=$cold timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02dw6_ab.txt; done
for pw in 256 2048; do echo "staged=83 pw=$pw $(GM_AB_DW_ONLY=1 GM_DOT_STAGED_PER_WARP=$pw timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02dw6_ab.txt; done
tail -1 $O/r02dw6_test.log; cat $O/r02dw6_ab.txt
