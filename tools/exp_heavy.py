"""Experiment: split of one C4 sum SpMM between the flat (light) and hub
kernels, and sensitivity to the hub threshold. Run each config in a fresh
process (env knobs are read once). Prints ms per call (L2 flushed)."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_16991_b200 as gm  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

red = {"sum": L.GM_SUM, "max": L.GM_MAX, "mean": L.GM_MEAN}[sys.argv[1] if len(sys.argv) > 1 else "sum"]
stream = torch.cuda.current_stream().cuda_stream
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, bench.F, "cuda", stream)
csc = g.to_csc()
plan = csc.plan()
cs = csc.c_struct()
out = torch.empty_like(x)
arg = torch.empty(x.shape, dtype=torch.int32, device="cuda") if red == L.GM_MAX else None
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def call():
    L.check(L.lib().gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), bench.F, None, None,
                            red, C.c_void_p(out.data_ptr()), None if arg is None else C.c_void_p(arg.data_ptr()),
                            C.c_void_p(stream)))


for _ in range(3):
    call()
ts = []
for _ in range(10):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    call()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
rp = csc.rowptr.cpu()
deg = rp[1:] - rp[:-1]
thr = plan.heavy_threshold
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("GM_")}, "ms": sum(ts) / len(ts),
                  "min_ms": min(ts), "heavy_rows": int(plan.num_heavy), "thr": int(thr),
                  "heavy_edges": int(deg[deg > thr].sum())}))
