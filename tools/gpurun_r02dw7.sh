# staged dw kernel, round 2: metadata one issue ahead, plain cp.async for cold rows; A/B + one --set full capture
O=gpurun_out
R=r02dw7
rm -f $O/${R}_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "edge_dot" > $O/${R}_test.log 2>&1; echo "pytest rc=$?" >> $O/${R}_test.log
for cfg in 0 83 44 162 46; do
  echo "staged=$cfg $(GM_AB_DW_ONLY=1 GM_DOT_STAGED=$cfg timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done
for cold in 0 1; do echo "staged=83 cold=$cold $(GM_AB_DW_ONLY=1 GM_DOT_STAGED_COLD=$cold timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/${R}_ab.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"edge_dot_staged" -c 1 -o $O/${R}_dw -f python tools/prof_edge_dot.py > $O/${R}_prof.log 2>&1
ncu -i $O/${R}_dw.ncu-rep --page raw --csv > $O/${R}_dw.raw.csv 2>/dev/null
ncu -i $O/${R}_dw.ncu-rep --page source --csv > $O/${R}_dw.src.csv 2>/dev/null; rm -f $O/${R}_dw.ncu-rep
tail -1 $O/${R}_test.log; cat $O/${R}_ab.txt
