O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layers.py -x -q -p no:cacheprovider -k "backward or dw or weight" > $O/r02n_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02n_gputest.log
for rep in 1 2; do
  echo "new $(python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02n_ab.txt
  echo "old $(GM_LIB_PATH=$PWD/paper_2507_16991_b200/libgraphmill_b200_old.so python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02n_ab.txt
done
tail -1 $O/r02n_gputest.log; cat $O/r02n_ab.txt
