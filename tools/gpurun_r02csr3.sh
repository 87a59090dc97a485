O=gpurun_out
rm -f $O/r02csr4_ab.txt
timeout 900 python -m pytest tests/test_gpu_csr_build.py tests/test_gpu_dist_build.py -x -q -p no:cacheprovider > $O/r02csr4_test.log 2>&1; echo "pytest rc=$?" >> $O/r02csr4_test.log
for rep in 1 2; do for v in base tm2 tm4 notma; do
  if [ $v = base ] || [ $v = notma ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  if [ $v = notma ]; then t=0; else t=1; fi
  echo "$v $(GM_RADIX_TMA=$t GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_csr.py 2>&1 | tail -1)" >> $O/r02csr4_ab.txt
done; done
tail -1 $O/r02csr4_test.log; cat $O/r02csr4_ab.txt
