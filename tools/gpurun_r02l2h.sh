# L2 hot-row budget (GM_L2_HOT_MB) re-checked after the CTA-size and window changes: headline step
O=gpurun_out
R=r02l2h
rm -f $O/${R}_ab.txt
for rep in 1 2; do for mb in 64 32 96 128; do
  GM_L2_HOT_MB=$mb timeout 900 python bench.py --no-cpu-baseline --no-secondary > $O/${R}_$mb.json 2> $O/${R}_$mb.err
  echo "hot_mb=$mb $(python -c "import json;d=json.load(open('$O/${R}_$mb.json'));print(d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
