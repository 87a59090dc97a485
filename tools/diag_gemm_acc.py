"""Accuracy profile of the fp32-operand segment_matmul (split-bf16 tcgen05
route) at the C1 layer-1 shape: error / S statistics (S = |x||W|) against fp64,
signed bias, and the same for K split into chunks (accumulation-depth check)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_16991_b200 as gm  # noqa: E402

rng = np.random.default_rng(0)
out = {}
for k, n in ((1433, 16), (1024, 16), (128, 128), (16, 16)):
    x = rng.uniform(-1, 1, (2708, k)).astype(np.float32)
    w = rng.uniform(-1 / np.sqrt(k), 1 / np.sqrt(k), (k, n)).astype(np.float32)
    ref = x.astype(np.float64) @ w.astype(np.float64)
    s = np.abs(x).astype(np.float64) @ np.abs(w).astype(np.float64)
    got = gm.segment_matmul(torch.from_numpy(x).cuda(), [0, 2708], torch.from_numpy(w).cuda()[None]).double().cpu().numpy()
    e = (got - ref) / s
    r32 = (x @ w).astype(np.float64)
    e32 = (r32 - ref) / s
    out[f"{k}x{n}"] = {"max_err_over_S": float(np.abs(e).max()), "mean_abs": float(np.abs(e).mean()),
                       "signed_mean": float(e.mean()), "norm_rel": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                       "numpy_f32_max": float(np.abs(e32).max()), "numpy_f32_norm_rel": float(np.linalg.norm(r32 - ref) / np.linalg.norm(ref))}
print(json.dumps(out))
