O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layers.py tests/test_gpu_hetero.py -x -q -p no:cacheprovider > $O/r02y_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02y_gputest.log
python - > $O/r02y_gemm.txt 2>&1 <<'PY'
import bench, torch
import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
for fp32 in (True, False):
    print(bench.bench_segment_matmul(gm, L, torch.device("cuda", 0), fp32=fp32))
PY
tail -3 $O/r02y_gputest.log; cat $O/r02y_gemm.txt
