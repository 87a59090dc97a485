"""Same-box A/B timing of build_compressed on the C4 graph's CSC (env knobs
read once per process): mean / min ms over 10 builds, L2 flushed between."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_16991_b200 as gm  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

stream = torch.cuda.current_stream()
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, 4, "cuda", stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
dst, src = g.dst(), g.src()
ref = gm.build_compressed(dst, src, bench.N_NODES)
per = bench.timed_steps(lambda: gm.build_compressed(dst, src, bench.N_NODES), 10, flush)
v = gm.build_compressed(dst, src, bench.N_NODES)
same = bool(torch.equal(v.perm, ref.perm) and torch.equal(v.col, ref.col) and torch.equal(v.rowptr, ref.rowptr))
def h(t):
    t = t.to(torch.int64)
    return int((t * torch.arange(1, t.numel() + 1, device=t.device, dtype=torch.int64) % 1000003).sum().item())
print(json.dumps({"env": {k: os.environ.get(k) for k in ("GM_CSR_ALGO", "GM_RADIX_BITS", "GM_CSR_ONESWEEP")},
                  "hash": [h(v.rowptr), h(v.col), h(v.perm)],
                  "ms": round(statistics.mean(per), 4), "min": round(min(per), 4), "repeatable": same}))
