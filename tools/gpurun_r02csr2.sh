O=gpurun_out
rm -f $O/r02csr2_ab.txt
for v in w4r8 w4r16 w2r16; do GM_LIB_PATH=$PWD/paper_2507_16991_b200/libgraphmill_b200_$v.so timeout 600 python -m pytest tests/test_gpu_csr_build.py -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/$v test /" >> $O/r02csr2_ab.txt; done
for rep in 1 2; do for v in base w4r8 w4r16 w2r16; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_csr.py 2>&1 | tail -1)" >> $O/r02csr2_ab.txt
done; done
cat $O/r02csr2_ab.txt
