# flat CTA size (GM_FLAT_THREADS) A/B on the headline step: 224 / 192 threads leave register room for a hub CTA
O=gpurun_out
R=r02ft2
rm -f $O/${R}_ab.txt
for rep in 1 2; do for t in 256 192 160 128 96; do
  GM_FLAT_THREADS=$t timeout 900 python bench.py --no-cpu-baseline --no-secondary > $O/${R}_$t.json 2> $O/${R}_$t.err
  echo "threads=$t $(python -c "import json;d=json.load(open('$O/${R}_$t.json'));print(d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
for t in 128; do GM_FLAT_THREADS=$t GM_PROF_SKIP=1 timeout 900 python bench.py --no-cpu-baseline --no-secondary > $O/${R}_flatonly_$t.json 2>/dev/null; echo "flat-only threads=$t $(python -c "import json;d=json.load(open('$O/${R}_flatonly_$t.json'));print(d['ms_per_step'])")" >> $O/${R}_ab.txt; done
cat $O/${R}_ab.txt
