"""Backward of the max / min aggregation path on B200:
aggregate's argpos scatter (aggregate.hpp:295-308) + the gather_rows adjoint
(tensor.hpp:510-524), against the reference tape (tests/golden/maxbwd.npz)
and the oracle restatement (pinned to that tape in tests/test_oracle.py).
Bar: dx bit-identical."""
import os

import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _run(src, dst, n, x, g, kind):
    e = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, n)
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    out, arg = gm.neighbor_aggregate(e, xt, kind, return_argmax=True)
    dx = gm.neighbor_aggregate_backward(e, kind, torch.from_numpy(np.ascontiguousarray(g)).cuda(), arg)
    torch.cuda.synchronize()
    return arg.cpu().numpy().astype(np.int64), dx.cpu().numpy()


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("kind", ["max", "min"])
def test_max_backward_matches_reference_tape(dt, kind):
    d = np.load(os.path.join(GOLD, "maxbwd.npz"))
    n = int(d["n"][0])
    arg, dx = _run(d["src"], d["dst"], n, d[f"{dt}_x"], d[f"{dt}_g"], kind)
    assert np.array_equal(arg, d[f"{dt}_{kind}_arg"])
    assert dx.tobytes() == d[f"{dt}_{kind}_dx"].tobytes()


@pytest.mark.parametrize("f,dtype", [(100, np.float32), (7, np.float32), (6, np.float32), (130, np.float32),
                                     (5, np.float64), (64, np.float64)])
def test_max_backward_vs_oracle_power_law(f, dtype):
    """Source hubs beyond the 1,024-entry threshold take the column-parallel
    hub kernel; widths select 16/8/4-byte lanes."""
    n, e = 6000, 400_000
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    L.lib().gm_synth_edges_host(1, 77 + f, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    rng = np.random.default_rng(f)
    x = (np.floor(rng.uniform(-1, 1, (n, f)) * 8) / 8).astype(dtype)  # ties everywhere
    g = rng.uniform(-1, 1, (n, f)).astype(dtype)
    orc = Oracle()
    rp, col, perm = orc.build_compressed(dst, src, n)
    assert np.bincount(src, minlength=n).max() > 1024
    for kind in ("max", "min"):
        arg, dx = _run(src, dst, n, x, g, kind)
        _, warg = orc.spmm_max(rp, col, perm, x, is_min=(kind == "min"))
        assert np.array_equal(arg, warg)
        want = orc.spmm_max_backward(rp, col, perm, warg, g, n)
        assert dx.tobytes() == want.tobytes()


def test_max_backward_edge_cases():
    # empty graph rows, an isolated source, duplicate edges, bipartite shapes
    src = np.array([0, 0, 2, 2, 2], np.int64)
    dst = np.array([1, 1, 3, 0, 3], np.int64)
    x = np.array([[1.0, -2.0], [5.0, 5.0], [1.0, 3.0]], np.float32)
    g = np.arange(8, dtype=np.float32).reshape(4, 2) + 1
    e = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), 3, 4)
    out, arg = gm.neighbor_aggregate(e, torch.from_numpy(x).cuda(), "max", return_argmax=True)
    dx = gm.neighbor_aggregate_backward(e, "max", torch.from_numpy(g).cuda(), arg).cpu().numpy()
    orc = Oracle()
    rp, col, perm = orc.build_compressed(dst, src, 4)
    _, warg = orc.spmm_max(rp, col, perm, x)
    assert np.array_equal(arg.cpu().numpy(), warg)
    assert dx.tobytes() == orc.spmm_max_backward(rp, col, perm, warg, g, 3).tobytes()
    with pytest.raises(ValueError):
        gm.neighbor_aggregate_backward(e, "sum", torch.from_numpy(g).cuda(), arg)


@pytest.mark.slow
def test_max_backward_full_c4_sampled_sources():
    """C4 shape (2.45M nodes, 61.9M edges, F=100): dx rows of sampled sources
    (random + the largest out-degree hubs) recomputed on the host from the COO
    arrays, independently of the source view: entries of s sorted by
    (destination, COO position), winners added in that order."""
    n, e_cnt, f = 2_449_029, 61_859_140, 100
    seed = 0x67726170686D696C
    s = torch.empty(e_cnt, dtype=torch.int64, device="cuda")
    d = torch.empty(e_cnt, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    L.check(L.lib().gm_synth_edges(1, seed, 0, e_cnt, n, n, s.data_ptr(), d.data_ptr(), stream))
    x = torch.empty(n, f, dtype=torch.float32, device="cuda")
    L.check(L.lib().gm_synth_features(seed, 0, n, f, 1, L.GM_F32, x.data_ptr(), stream))
    gen = torch.Generator(device="cuda").manual_seed(5)
    g = torch.rand(n, f, device="cuda", generator=gen) * 2 - 1
    ei = gm.EdgeIndex(s, d, n, n)
    _, arg = gm.neighbor_aggregate(ei, x, "max", return_argmax=True)
    dx = gm.neighbor_aggregate_backward(ei, "max", g, arg)
    outdeg = torch.bincount(s, minlength=n)
    rows = torch.unique(torch.cat([torch.topk(outdeg, 12).indices,
                                   torch.randint(0, n, (600,), device="cuda", generator=gen)]))
    mark = torch.zeros(n, dtype=torch.bool, device="cuda")
    mark[rows] = True
    pos = torch.nonzero(mark[s]).flatten()
    ps, pd = s[pos].cpu().numpy(), d[pos].cpu().numpy()
    pos = pos.cpu().numpy()
    argh = arg[torch.from_numpy(pd).cuda()].cpu().numpy()
    gh = g[torch.from_numpy(pd).cuda()].cpu().numpy()
    got = dx[rows].cpu().numpy()
    order = np.lexsort((pos, pd, ps))  # by source, then destination, then COO position
    want = {int(r): np.zeros(f, np.float32) for r in rows.cpu().numpy()}
    for i in order:
        acc = want[int(ps[i])]
        hit = argh[i] == pos[i]
        acc[hit] = acc[hit] + gh[i][hit]
    for k, r in enumerate(rows.cpu().numpy()):
        assert got[k].tobytes() == want[int(r)].tobytes(), f"source {r}"
