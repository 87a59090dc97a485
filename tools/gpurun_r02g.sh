O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr_build.py -x -q -p no:cacheprovider > $O/r02j_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02j_gputest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02j_csr.csv python tools/prof_csr.py --iters 1 > $O/r02j_csr.log 2>&1
for rep in 1 2; do for v in base m16 m8b r8b m12; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_csr.py 2>&1 | tail -1)" >> $O/r02j_ab.txt
done; done
tail -2 $O/r02j_gputest.log; cat $O/r02j_ab.txt
