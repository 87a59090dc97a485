O=gpurun_out
rm -f $O/r02dw_ab.txt
GM_LIB_PATH=$PWD/paper_2507_16991_b200/libgraphmill_b200_gs.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "backward or dw or weight" > $O/r02dw_test.log 2>&1; echo "pytest rc=$?" >> $O/r02dw_test.log
for rep in 1 2; do for v in base gs; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  echo "$v $(GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02dw_ab.txt
done; done
tail -1 $O/r02dw_test.log; cat $O/r02dw_ab.txt
