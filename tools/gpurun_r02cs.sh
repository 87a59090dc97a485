# CSR radix: column-scan walk with 8 rows in flight — same-box A/B vs the previous build + launch list (hashes must match)
O=gpurun_out
R=r02cs
rm -f $O/${R}_ab.txt
timeout 600 python -m pytest tests/test_gpu_csr_build.py -x -q -p no:cacheprovider > $O/${R}_test.log 2>&1; echo "pytest rc=$?" >> $O/${R}_test.log
for rep in 1 2; do for v in base prev; do
  if [ "$v" = base ]; then lib=paper_2507_16991_b200/libgraphmill_b200.so; else lib=paper_2507_16991_b200/libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/$lib timeout 300 python tools/ab_csr.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"radix_col" -c 9 --log-file $O/${R}_launches.csv python tools/prof_csr.py --iters 1 > $O/${R}_ncu.log 2>&1
tail -1 $O/${R}_test.log; cat $O/${R}_ab.txt
