# dw tile kernel: parity tests + same-box A/B (slice vs tile T=32/16, MINB variants)
set -x
O=gpurun_out
R=r02u2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "edge_dot or backward" > $O/${R}_test.log 2>&1; echo "rc=$?" >> $O/${R}_test.log
for i in 1 2; do
GM_EDGE_DOT_TILE=0 timeout 300 python tools/ab_backward.py > $O/${R}_slice_$i.json 2>&1
timeout 300 python tools/ab_backward.py > $O/${R}_t32_$i.json 2>&1
for v in t16 t16m3 t32m3; do GM_LIB_PATH=paper_2507_16991_b200/libgraphmill_b200_$v.so timeout 300 python tools/ab_backward.py > $O/${R}_${v}_$i.json 2>&1; done
done
tail -3 $O/${R}_test.log; for f in $O/${R}_*.json; do echo $f $(tail -1 $f); done
