# flat CTA size: C5 papers100M-shaped bf16 line (256 vs 128) + the full GPU suite and smoke on the new default
O=gpurun_out
R=r02ft5
rm -f $O/${R}_ab.txt
for t in 256 128; do
  GM_FLAT_THREADS=$t GM_AB_HASH=1 timeout 1200 python tools/bench_configs.py C5 > $O/${R}_c5_$t.log 2>&1
  echo "threads=$t $(grep '"reduce"' $O/${R}_c5_$t.log | tr '\n' ' ') $(tail -2 $O/${R}_c5_$t.log | grep -i error | head -1)" >> $O/${R}_ab.txt
done


cat $O/${R}_ab.txt; tail -3 $O/${R}_gputest.log
