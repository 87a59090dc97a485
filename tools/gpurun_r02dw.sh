O=gpurun_out
rm -f $O/r02dw5_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -p no:cacheprovider -k "backward or dw or weight or empty or slice" > $O/r02dw5_test.log 2>&1; echo "pytest rc=$?" >> $O/r02dw5_test.log
for rep in 1 2; do for p in 1 0; do
  echo "pipe=$p $(GM_EDGE_DOT_PIPE=$p python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02dw5_ab.txt
done; done
tail -1 $O/r02dw5_test.log; cat $O/r02dw5_ab.txt
