# headline decomposition: flat-only (GM_PROF_SKIP=1) and hub-only (=2) steps vs the full call (bench timing, no CPU baseline)
O=gpurun_out
R=r02hub
rm -f $O/${R}_ab.txt
for rep in 1 2; do for sk in 0 1 2; do
  GM_PROF_SKIP=$sk timeout 900 python bench.py --no-cpu-baseline --no-secondary > $O/${R}_s$sk.json 2> $O/${R}_s$sk.err
  echo "skip=$sk $(python -c "import json;d=json.load(open('$O/${R}_s$sk.json'));print(d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
