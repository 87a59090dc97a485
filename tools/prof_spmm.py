"""Profiling driver: the bench workload's SpMM (C4 products-shaped, F=100 fp32)
run `--iters` times after setup. Use under ncu (never a bench number)."""
import argparse
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_16991_b200 as gm  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--reduce", default="sum")
ap.add_argument("--f", type=int, default=bench.F)
args = ap.parse_args()
stream = torch.cuda.current_stream().cuda_stream
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, args.f, "cuda", stream)
csc = g.to_csc()
plan = csc.plan()
cs = csc.c_struct()
out = torch.empty_like(x)
arg = torch.empty(x.shape, dtype=torch.int32, device="cuda") if args.reduce in ("max", "min") else None
red = {"sum": L.GM_SUM, "mean": L.GM_MEAN, "max": L.GM_MAX, "min": L.GM_MIN}[args.reduce]
torch.cuda.synchronize()
for _ in range(args.iters):
    L.check(L.lib().gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), args.f, None,
                            None, red, C.c_void_p(out.data_ptr()),
                            None if arg is None else C.c_void_p(arg.data_ptr()), C.c_void_p(stream)))
torch.cuda.synchronize()
print("heavy rows", plan.num_heavy, "windows", plan.num_windows)
