# flat CTA size 128 (new default) vs 256 across the bench's lines and the per-config SpMM lines (C2, C5, C3 relation)
O=gpurun_out
R=r02ft3
rm -f $O/${R}_ab.txt
for t in 256 128; do
  GM_FLAT_THREADS=$t timeout 900 python bench.py --no-cpu-baseline > $O/${R}_$t.json 2> $O/${R}_$t.err
  echo "threads=$t $(python -c "
import json;d=json.load(open('$O/${R}_$t.json'));s=d['secondary']
print(d['ms_per_step'], d['e2e']['ms_per_step'], {k:round(v['ms'],3) for k,v in s.items() if isinstance(v,dict) and 'ms' in v})" 2>&1 | tail -1)" >> $O/${R}_ab.txt
  echo "threads=$t $(GM_FLAT_THREADS=$t GM_AB_HASH=1 timeout 900 python tools/bench_configs.py C2 C5 C3 2>&1 | grep '"reduce"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['reduce'], round(d['ms'],3), d.get('out_hash'))" | tr '\n' ';')" >> $O/${R}_ab.txt
done
cat $O/${R}_ab.txt
