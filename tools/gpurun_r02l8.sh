# fp32 hub kernel with 8-byte lanes (half the CTAs per hub row): parity tests with hubs + same-box A/B on the headline and max lines
O=gpurun_out
R=r02l8
rm -f $O/${R}_ab.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edge_cases.py tests/test_gpu_dist_push.py tests/test_gpu_dist_blocked.py -x -q -p no:cacheprovider > $O/${R}_test.log 2>&1; echo "pytest rc=$?" >> $O/${R}_test.log
for rep in 1 2; do for v in lane8 lane4 lane8ring8; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; extra=""
  case $v in lane4) extra="GM_HUB_LANE8=0";; lane8ring8) lib=paper_2507_16991_b200/libgraphmill_b200_ring8.so;; esac
  env GM_LIB_PATH=$PWD/$lib $extra timeout 900 python bench.py --no-cpu-baseline > $O/${R}_$v.json 2> $O/${R}_$v.err
  echo "$v $(python -c "import json;d=json.load(open('$O/${R}_$v.json'));print(d['ms_per_step'], d['roofline']['frac'], d['secondary']['max_argmax_spmm']['ms'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
for v in lane8 lane4; do extra=""; [ $v = lane4 ] && extra="GM_HUB_LANE8=0"; env $extra GM_PROF_SKIP=2 timeout 900 python bench.py --no-cpu-baseline --no-secondary > $O/${R}_hubonly_$v.json 2>/dev/null; echo "hub-only $v $(python -c "import json;d=json.load(open('$O/${R}_hubonly_$v.json'));print(d['ms_per_step'])")" >> $O/${R}_ab.txt; done
tail -1 $O/${R}_test.log; cat $O/${R}_ab.txt
