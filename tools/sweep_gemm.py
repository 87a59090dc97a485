"""segment_matmul throughput: C3 (OGB-MAG) shape and an F-sweep (K = N = F)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json  # noqa: E402

import paper_2507_16991_b200 as gm  # noqa: E402

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
res = []
for f, rows in ((128, 1_939_743), (256, 1_939_743), (512, 1_000_000), (1024, 500_000), (2048, 262_144)):
    ptr = [0, rows * 38 // 100, rows * 96 // 100, rows * 97 // 100, rows]
    x = torch.randn(rows, f, device="cuda").to(torch.bfloat16)
    w = (torch.randn(4, f, f, device="cuda") / f ** 0.5).to(torch.bfloat16)
    for _ in range(3):
        gm.segment_matmul(x, ptr, w)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        gm.segment_matmul(x, ptr, w)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    flops = 2.0 * rows * f * f
    byts = 2.0 * rows * f * 2 + 4 * f * f * 2
    r = {"F": f, "rows": rows, "ms": ms, "tflops": flops / ms / 1e9, "frac_tensor": flops / ms / 1e9 / peaks["bf16_tflops"],
         "gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / peaks["hbm_gbs"]}
    res.append(r)
    print(json.dumps(r))
