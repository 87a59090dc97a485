O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist_blocked.py -x -q -p no:cacheprovider > $O/r02hub_test.log 2>&1; echo "pytest rc=$?" >> $O/r02hub_test.log
for rep in 1 2; do for v in base prehub; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_flat.py 2>&1 | tail -1)" >> $O/r02hub_ab.txt
done; done
GM_PROF_SKIP=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02hub_launch.csv python tools/prof_spmm.py --iters 1 > /dev/null 2>&1
tail -2 $O/r02hub_test.log; cat $O/r02hub_ab.txt; grep hub $O/r02hub_launch.csv | awk -F'","' '{print $NF}'
