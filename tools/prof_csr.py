"""Profiling driver: build_compressed of the bench graph's CSC (C4 products
shape), `--iters` fresh builds after setup. Use under ncu (never a bench number)."""
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
stream = torch.cuda.current_stream().cuda_stream
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, 4, "cuda", stream)
torch.cuda.synchronize()
for _ in range(args.iters):
    v = gm.build_compressed(g.dst(), g.src(), bench.N_NODES, bench.N_NODES)
torch.cuda.synchronize()
print("nnz", v.num_entries())
