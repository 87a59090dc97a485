O=gpurun_out
rm -f $O/r02mb_ab.txt
#GM_MAXBWD_STAGED=1 timeout 600 python -m pytest tests/test_gpu_maxbwd.py tests/test_gpu_edge_cases.py -x -q -p no:cacheprovider > $O/r02mb_test.log 2>&1; echo "pytest rc=$?" >> $O/r02mb_test.log
for rep in 1 2; do for v in s2w4 s2w2 s3w2 s4w4; do
  if [ $v = base ]; then lib=libgraphmill_b200.so; else lib=libgraphmill_b200_$v.so; fi
  if [ $v = base ]; then st=0; else st=1; fi
  echo "$v $(GM_MAXBWD_STAGED=$st GM_LIB_PATH=$PWD/paper_2507_16991_b200/$lib python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02mb_ab.txt
done; done
tail -1 $O/r02mb_test.log; cat $O/r02mb_ab.txt
