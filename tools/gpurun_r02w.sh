# Final evidence pass on HEAD (CTA size + window size changes): GPU tests, smoke, bench (both arms), contract launch list,
# --set full of the headline flat kernel (sum) and the max flat kernel.
set -x
O=gpurun_out
R=r02w
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${R}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${R}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1
timeout 900 python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_ref.json 2> $O/${R}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/${R}_bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spmm_flat|spmm_hub" -c 2 -o $O/${R}_spmm -f python tools/prof_spmm.py --iters 1 >> $O/${R}_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spmm_flat|spmm_hub" -c 2 -o $O/${R}_max -f python tools/prof_spmm.py --iters 1 --reduce max >> $O/${R}_prof.log 2>&1
for r in spmm max; do ncu -i $O/${R}_$r.ncu-rep --page raw --csv > $O/${R}_$r.raw.csv 2>/dev/null; rm -f $O/${R}_$r.ncu-rep; done
du -sh $O
tail -2 $O/${R}_gputest.log; tail -1 $O/${R}_smoke.log; cat $O/${R}_bench.json | head -c 600
