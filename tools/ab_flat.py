"""Same-box A/B timing of the C4 flat SpMM variants (env knobs such as
GM_FLAT_LM3 / GM_FLAT_MAX_U are read once per process): prints one JSON line
with the mean per-call ms of sum and max+argmax, L2 flushed between calls."""
import ctypes as C
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
g, x = bench.make_graph(gm, L, bench.N_NODES, bench.N_EDGES, bench.F, "cuda", stream.cuda_stream)
csc = g.to_csc()
plan = csc.plan()
cs = csc.c_struct()
out = torch.empty_like(x)
arg = torch.empty(x.shape, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {k: os.environ.get(k) for k in ("GM_FLAT_LM3", "GM_FLAT_MAX_U")}
for name, red, a in (("sum", L.GM_SUM, None), ("max", L.GM_MAX, arg)):
    def step():
        L.check(L.lib().gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), bench.F, None, None,
                                red, C.c_void_p(out.data_ptr()), None if a is None else C.c_void_p(a.data_ptr()),
                                C.c_void_p(stream.cuda_stream)))
    for _ in range(3):
        step()
    per = bench.timed_steps(step, 20, flush)
    res[name] = round(statistics.mean(per), 4)
    res[name + "_min"] = round(min(per), 4)
torch.cuda.synchronize()
print(json.dumps(res))
