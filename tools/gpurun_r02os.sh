# one-sweep radix CSR build: CSR parity tests + same-box A/B (hashes must match) + launch list
O=gpurun_out
R=r02os
rm -f $O/${R}_ab.txt
timeout 900 python -m pytest tests/test_gpu_csr_build.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist_build.py tests/test_gpu_edge_cases.py tests/test_gpu_edge_index.py -x -q -p no:cacheprovider > $O/${R}_test.log 2>&1; echo "pytest rc=$?" >> $O/${R}_test.log
for rep in 1 2; do for os in 0 1; do
  echo "onesweep=$os $(GM_CSR_ONESWEEP=$os timeout 300 python tools/ab_csr.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"radix|rowptr_from" -c 12 --log-file $O/${R}_launches.csv python tools/prof_csr.py --iters 1 > $O/${R}_ncu.log 2>&1
tail -1 $O/${R}_test.log; cat $O/${R}_ab.txt
