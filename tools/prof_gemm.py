"""Profiling driver: C3 (OGB-MAG) segment_matmul, K=N=128 bf16 (or fp32 operands with
`--fp32`: the fused-split kernel), `--iters` calls."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_16991_b200 as gm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--f", type=int, default=128)
ap.add_argument("--fp32", action="store_true")
args = ap.parse_args()
ptr = [0, 736_389, 1_871_038, 1_879_778, 1_939_743]
x = torch.randn(ptr[-1], args.f, device="cuda").to(torch.bfloat16)
w = (torch.randn(4, args.f, args.f, device="cuda") / 11).to(torch.bfloat16)
if args.fp32:
    x, w = x.float(), w.float()
for _ in range(args.iters):
    gm.segment_matmul(x, ptr, w)
torch.cuda.synchronize()
