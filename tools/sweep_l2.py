"""Sweep the SpMM L2 hot-row budget (plan.l2_hot_bytes) on the bench workload.
Each timed call is preceded by a 256 MB L2 flush (outside the events)."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_16991_b200 as gm  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

stream = torch.cuda.current_stream().cuda_stream
f = int(sys.argv[1]) if len(sys.argv) > 1 else bench.F
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, f, "cuda", stream)
csc = g.to_csc()
plan = csc.plan()
cs = csc.c_struct()
out = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for red_name, red in (("sum", L.GM_SUM), ("max", L.GM_MAX)):
    for mb in (0, 16, 32, 48, 64, 80, 96, 112):
        plan.l2_hot_bytes = mb << 20
        times = []
        for it in range(8):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            L.check(L.lib().gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), f, None,
                                    None, red, C.c_void_p(out.data_ptr()), None, C.c_void_p(stream)))
            b.record()
            torch.cuda.synchronize()
            if it >= 3:
                times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        print(f"{red_name} f={f} hot={mb:4d} MB  {ms:7.3f} ms  {bench.N_EDGES / ms / 1e6:6.2f} GEdges/s")
