# Round-2 evidence pass: GPU tests, smoke, bench (both arms), the contract's ncu
# launch list of the bench command, --set full captures of the top kernels.
set -x
O=gpurun_out
R=r02f
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${R}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${R}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1
timeout 900 python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_ref.json 2> $O/${R}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/${R}_bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm_(flat|hub)_kernel" -c 2 -o $O/${R}_spmm_sum -f python tools/prof_spmm.py --iters 1 > $O/${R}_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm_(flat|hub)_kernel" -c 2 -o $O/${R}_spmm_max -f python tools/prof_spmm.py --reduce max --iters 1 >> $O/${R}_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"radix|rowptr_from" -c 20 -o $O/${R}_csr -f python tools/prof_csr.py --iters 1 >> $O/${R}_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"edge_dot_csc_v4" -c 1 -o $O/${R}_dw -f python tools/prof_edge_dot.py >> $O/${R}_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"maxbwd" -c 2 -o $O/${R}_maxbwd -f python tools/prof_maxbwd.py --iters 1 >> $O/${R}_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"segment_matmul_kernel" -c 1 -o $O/${R}_gemm_fp32 -f python tools/prof_gemm.py --fp32 --iters 1 >> $O/${R}_prof.log 2>&1
for r in spmm_sum spmm_max csr dw maxbwd gemm_fp32; do ncu -i $O/${R}_$r.ncu-rep --page raw --csv > $O/${R}_$r.raw.csv 2>/dev/null; rm -f $O/${R}_$r.ncu-rep; done
du -sh $O
tail -2 $O/${R}_gputest.log; tail -1 $O/${R}_smoke.log
