# e2e over K steps + hub-threshold A/B of the headline (bench lines, no CPU baseline)
O=gpurun_out
R=r02e2e
rm -f $O/${R}_ab.txt
for thr in 1024 512 2048 1024; do
  GM_HEAVY_THR=$thr timeout 900 python bench.py --no-cpu-baseline > $O/${R}_thr$thr.json 2> $O/${R}_thr$thr.err
  echo "thr=$thr $(python -c "import json;d=json.load(open('$O/${R}_thr$thr.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step'], d['plan'] if 'plan' in d else '')")" >> $O/${R}_ab.txt
done
cat $O/${R}_ab.txt
