# max backward: skip the cp.async of non-matching gradient slices (was: zero-fill copies) — tests + same-box A/B + DRAM bytes
O=gpurun_out
R=r02mz
rm -f $O/${R}_ab.txt
timeout 900 python -m pytest tests/test_gpu_maxbwd.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "max or backward" > $O/${R}_test.log 2>&1; echo "pytest rc=$?" >> $O/${R}_test.log
for rep in 1 2; do for v in base zfill; do
  if [ "$v" = base ]; then lib=paper_2507_16991_b200/libgraphmill_b200.so; else lib=paper_2507_16991_b200/libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/$lib timeout 300 python tools/ab_backward.py 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
for v in base zfill; do
  if [ "$v" = base ]; then lib=paper_2507_16991_b200/libgraphmill_b200.so; else lib=paper_2507_16991_b200/libgraphmill_b200_$v.so; fi
  GM_LIB_PATH=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"maxbwd" --log-file $O/${R}_${v}_launches.csv python tools/prof_maxbwd.py > $O/${R}_${v}_ncu.log 2>&1
done
tail -1 $O/${R}_test.log; cat $O/${R}_ab.txt
