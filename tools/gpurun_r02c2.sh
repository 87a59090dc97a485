# C2 Reddit-shaped (F=602 fp32): hub-row threshold for wide rows (4096 base; GM_HEAVY_THR raises it), mean and max lines
O=gpurun_out
R=r02c2
rm -f $O/${R}_ab.txt
for thr in 0 8192 16384; do
  extra=""; [ $thr != 0 ] && extra="GM_HEAVY_THR=$thr"
  echo "thr=$thr $(env $extra GM_AB_HASH=1 timeout 900 python tools/bench_configs.py C2 C2X 2>&1 | grep '"reduce"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['reduce'], round(d['ms'],3), d['heavy_rows'], d.get('out_hash'))" | tr '\n' ';')" >> $O/${R}_ab.txt
done
cat $O/${R}_ab.txt
