"""Profiling driver: max/min aggregation backward (gm_spmm_max_backward over
the cached source view) on the C4 graph, `--iters` calls after setup. Use
under ncu (never a bench number)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_16991_b200 as gm  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2)
args = ap.parse_args()
stream = torch.cuda.current_stream()
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, bench.F, "cuda", stream.cuda_stream)
gout = torch.rand_like(x)
_, arg = gm.neighbor_aggregate(g, x, "max", return_argmax=True)
gm.neighbor_aggregate_backward(g, "max", gout, arg)  # builds the source view once
torch.cuda.synchronize()
for _ in range(args.iters):
    gm.neighbor_aggregate_backward(g, "max", gout, arg)
torch.cuda.synchronize()
