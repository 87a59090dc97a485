O=gpurun_out
rm -f $O/r02mb3_ab.txt
timeout 600 python -m pytest tests/test_gpu_maxbwd.py tests/test_gpu_edge_cases.py -x -q -p no:cacheprovider > $O/r02mb3_test.log 2>&1; echo "pytest rc=$?" >> $O/r02mb3_test.log
for rep in 1 2; do for h in 1; do
echo "hot=$h $(GM_MAXBWD_HOT=$h python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02mb3_ab.txt
done; done
tail -1 $O/r02mb3_test.log; cat $O/r02mb3_ab.txt
