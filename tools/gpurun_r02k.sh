O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layers.py tests/test_gpu_csr_build.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > $O/r02l_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02l_gputest.log
for rep in 1 2; do
  echo "v4 $(python tools/ab_backward.py 2>&1 | tail -1)" >> $O/r02l_ab.txt
done
python tools/ab_csr.py >> $O/r02l_ab.txt 2>&1
ncu --set full --clock-control none -k regex:"edge_dot_csc_v4" -c 1 -o $O/r02l_v4 -f python tools/prof_edge_dot.py > $O/r02l_dot.log 2>&1
ncu -i $O/r02l_v4.ncu-rep --page raw --csv > $O/r02l_v4.raw.csv 2>/dev/null
tail -2 $O/r02l_gputest.log; cat $O/r02l_ab.txt
