"""Profiling driver: one BASELINE config's SpMM run `--iters` times after
setup (use under ncu; never a bench number).
  python tools/prof_config.py C5|C2|C4 [--iters 2] [--reduce sum]"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench_configs as bc  # noqa: E402
import paper_2507_16991_b200 as gm  # noqa: E402

CFG = {"C4": (1, 2_449_029, 61_859_140, 100, torch.float32), "C2": (1, 232_965, 114_615_892, 602, torch.float32),
       "C5": (1, 111_059_956, 1_615_685_872, 128, torch.bfloat16)}
ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--reduce", default="sum")
a = ap.parse_args()
kind, n, e, f, dt = CFG[a.config]
g = bc.graph(kind, n, e)
x = bc.feats(n, f, dt)
g.to_csc().plan(row_bytes=f * x.element_size())
torch.cuda.synchronize()
for _ in range(a.iters):
    if a.reduce in ("max", "min"):
        gm.neighbor_aggregate(g, x, a.reduce, return_argmax=True)
    else:
        gm.spmm(g, x, None, a.reduce)
torch.cuda.synchronize()
