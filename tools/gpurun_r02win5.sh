# auto window size (1024 with an 8-wave floor; 256 for >= 1 KB rows): bench lines, per-config lines (hashes), full GPU suite, smoke
O=gpurun_out
R=r02win5
rm -f $O/${R}_ab.txt
timeout 900 python bench.py --no-cpu-baseline > $O/${R}_bench.json 2> $O/${R}_bench.err
echo "bench $(python -c "import json;d=json.load(open('$O/${R}_bench.json'));s=d['secondary'];print(d['ms_per_step'], d['roofline']['frac'], {k:round(v['ms'],3) for k,v in s.items() if isinstance(v,dict) and 'ms' in v})" 2>&1 | tail -1)" >> $O/${R}_ab.txt
echo "configs $(GM_AB_HASH=1 timeout 1500 python tools/bench_configs.py C3 C2 C2X C5 2>&1 | grep '"reduce"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['reduce'], round(d['ms'],3), d.get('out_hash'))" | tr '\n' ';')" >> $O/${R}_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${R}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${R}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O/${R}_gputest.log 2>&1
cat $O/${R}_ab.txt; tail -3 $O/${R}_gputest.log
