# round-2 profiling pass: launch lists (contract pass) + --set full captures
set -x
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02b_csr_launches.csv python tools/prof_csr.py --iters 2 > $O/r02b_csr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"radix|rowptr_from|scan32" --launch-skip 0 -c 12 -o $O/r02b_csr_full -f python tools/prof_csr.py --iters 2 >> $O/r02b_csr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm_flat_kernel" -c 1 -o $O/r02b_flat_max -f python tools/prof_spmm.py --reduce max --iters 1 > $O/r02b_max.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"edge_dot_csc" -c 1 -o $O/r02b_edge_dot -f python tools/prof_edge_dot.py > $O/r02b_dot.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02b_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-secondary > $O/r02b_bench_ncu.log 2>&1
for r in r02b_csr_full r02b_flat_max r02b_edge_dot; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null; done
ls -la $O
