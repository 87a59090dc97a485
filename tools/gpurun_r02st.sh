# CSR radix: intermediate-pass store policy (streaming vs default) and 16-round tiles, same-box A/B (hashes must match)
O=gpurun_out
R=r02st
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base nostcs r16; do
  if [ "$v" = base ]; then lib=paper_2507_16991_b200/libgraphmill_b200.so; else lib=paper_2507_16991_b200/libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/$lib timeout 300 python tools/ab_csr.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
GM_LIB_PATH=$PWD/paper_2507_16991_b200/libgraphmill_b200_nostcs.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"radix_scatter" -c 3 --log-file $O/${R}_nostcs_launches.csv python tools/prof_csr.py --iters 1 > $O/${R}_ncu.log 2>&1
cat $O/${R}_ab.txt
