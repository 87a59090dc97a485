"""Profiling driver: gm_edge_dot on the C4 graph (use under ncu)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench_configs as bc  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

n, e, f = 2_449_029, 61_859_140, 100
g = bc.graph(1, n, e)
x = bc.feats(n, f, torch.float32)
gout = bc.feats(n, f, torch.float32)
dw = torch.empty(e, device="cuda")
for _ in range(2):
    L.check(L.lib().gm_edge_dot(L.GM_F32, g.src().data_ptr(), g.dst().data_ptr(), e, gout.data_ptr(), x.data_ptr(), f,
                                dw.data_ptr(), torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()

# the CSC-order kernel spmm_backward uses (gm_edge_dot_csc)
import ctypes as C  # noqa: E402
csc = g.to_csc()
cs = csc.c_struct()
rows = csc.entry_rows()
for _ in range(2):
    L.check(L.lib().gm_edge_dot_csc(L.GM_F32, C.byref(cs), C.byref(csc.plan()), rows.data_ptr(), gout.data_ptr(), x.data_ptr(), f,
                                    dw.data_ptr(), torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
