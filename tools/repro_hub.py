"""Medium power-law graph through gm_spmm (flat + hub kernels), checked
against the oracle. Debug aid for the hub kernel."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from oracle.oracle import Oracle
n, e, f = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
lib = L.lib()
src = np.zeros(e, np.int64); dst = np.zeros(e, np.int64)
lib.gm_synth_edges_host(1, 5, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
x = np.zeros((n, f), np.float32)
lib.gm_synth_features_host(5, 0, n, f, 1, L.GM_F32, x.ctypes.data)
g = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, n)
xt = torch.from_numpy(x).cuda()
for it in range(3):
    out = gm.spmm(g, xt, None, "sum")
    torch.cuda.synchronize()
print("heavy", g.to_csc().plan().num_heavy)
orc = Oracle()
rp, col, perm = orc.build_compressed(dst, src, n)
want = orc.spmm(rp, col, perm, x)
print("sum bit-exact:", out.cpu().numpy().tobytes() == want.tobytes())
