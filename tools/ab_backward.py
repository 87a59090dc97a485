"""Same-box timing of the C4 backward kernels (L2 flushed between calls):
dw (gm_edge_dot_csc, with / without the plan's L2 residency classes) and the
max/min backward gather (gm_spmm_max_backward)."""
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
torch.manual_seed(0)
gout = torch.rand_like(x)
csc = g.to_csc()
plan = csc.plan(400)
cs = csc.c_struct()
rows = csc.entry_rows()
dw = torch.empty(bench.N_EDGES, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, pl in (("dw_hint", C.byref(plan)), ("dw_nohint", None)):
    def step():
        L.check(L.lib().gm_edge_dot_csc(L.GM_F32, C.byref(cs), pl, rows.data_ptr(), gout.data_ptr(), x.data_ptr(),
                                        bench.F, dw.data_ptr(), C.c_void_p(stream.cuda_stream)))
    per = bench.timed_steps(step, 10, flush)
    res[name] = round(statistics.mean(per), 4)
    bits = dw.view(torch.int32).to(torch.int64)
    res[name + "_hash"] = int((bits * torch.arange(1, bits.numel() + 1, device="cuda", dtype=torch.int64) % 1000003).sum().item())
if os.environ.get("GM_AB_DW_ONLY"):
    print(json.dumps(res))
    sys.exit(0)
_, arg = gm.neighbor_aggregate(g, x, "max", return_argmax=True)
gm.neighbor_aggregate_backward(g, "max", gout, arg)
per = bench.timed_steps(lambda: gm.neighbor_aggregate_backward(g, "max", gout, arg), 10, flush)
res["max_backward"] = round(statistics.mean(per), 4)
print(json.dumps(res))
