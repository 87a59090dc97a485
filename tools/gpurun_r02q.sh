O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxbwd.py -x -q -p no:cacheprovider > $O/r02t_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02t_gputest.log
for rep in 1 2; do for v in base u6 u4b3; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02t_ab.txt
done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02t_mb.csv python tools/prof_maxbwd.py --iters 1 > $O/r02t.log 2>&1
tail -2 $O/r02t_gputest.log; cat $O/r02t_ab.txt
