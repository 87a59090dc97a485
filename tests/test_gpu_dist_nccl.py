"""gm_dist_spmm (the multi-GPU C-ABI over NCCL) on one B200 with a 1-rank
communicator: the NCCL plumbing (unique id, communicator, all-gather /
send-recv on the comm stream, device events gating the blocks) runs for real;
with one rank every source is in the own shard, so all three modes must equal
the single-GPU gm_spmm bit for bit (bf16 sum/mean through the fp32 carry: one
rounding per row, as on one GPU). Multi-rank block logic is covered by the
virtual-rank tests (test_gpu_dist_blocked.py) and the gloo tests."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from paper_2507_16991_b200.dist import DistSpmm, NcclComm, chunk_layout

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = NcclComm(0, 1)
    yield c
    c.close()


def graph(n=20000, e=400_000, seed=3):
    s = torch.empty(e, dtype=torch.int64, device="cuda")
    d = torch.empty(e, dtype=torch.int64, device="cuda")
    L.check(L.lib().gm_synth_edges(1, seed, 0, e, n, n, s.data_ptr(), d.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
    return gm.EdgeIndex(s, d, n, n)


@pytest.mark.parametrize("mode", ["exact", "blocked", "halo"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_one_rank_modes_equal_single_gpu(comm, mode, dtype):
    n = 20000
    g = graph(n)
    csc = g.to_csc()
    f = 64
    x = (torch.rand(n, f, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) * 2 - 1)
    x = (torch.floor(x * 8) / 8).to(dtype)  # ties for max/min
    kw = {}
    if mode == "halo":
        empty = torch.empty(0, dtype=torch.int32, device="cuda")
        kw = dict(need=[empty], send=[empty])
    ds = DistSpmm(csc, n, comm, mode=mode, chunks=4, **kw)
    if mode == "blocked":
        s_rows, cs = chunk_layout(n, 1, 4)
        xs = torch.zeros(4 * cs, f, dtype=dtype, device="cuda")
        xs[:n] = x
    else:
        xs = x
    for reduce in ("sum", "mean", "max", "min"):
        if reduce in ("sum", "mean"):
            want = gm.neighbor_aggregate(g, x, reduce)
            got = ds(xs, reduce)
            torch.cuda.synchronize()
            assert torch.equal(got.view(torch.uint8) if dtype == torch.bfloat16 else got,
                               want.view(torch.uint8) if dtype == torch.bfloat16 else want), (mode, reduce)
        else:
            want, warg = gm.neighbor_aggregate(g, x, reduce, return_argmax=True)
            got, arg = ds(xs, reduce)
            torch.cuda.synchronize()
            assert torch.equal(arg, warg), (mode, reduce)
            assert torch.equal(got.float(), want.float()), (mode, reduce)
    # repeat calls reuse the workspace and the events
    a = ds(xs, "max")[0]
    b = ds(xs, "max")[0]
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_layout_validation(comm):
    n = 1000
    g = graph(n, 20000)
    ds = DistSpmm(g.to_csc(), n, comm, mode="blocked", chunks=2)
    s_rows, cs = chunk_layout(n, 1, 2)
    xs = torch.zeros(2 * cs, 8, device="cuda")
    with pytest.raises(ValueError):
        L.check(L.lib().gm_dist_spmm(None, L.GM_F32, xs.data_ptr(), 8, L.GM_SUM, xs.data_ptr(), None, None, 0,
                                     comm.comm, None, None))
    # max/min in blocked mode need the argmax carry
    import ctypes as C
    ds.layout.plans = ds._plans_for(32)
    out = torch.empty(n, 8, device="cuda")
    with pytest.raises(ValueError):
        L.check(L.lib().gm_dist_spmm(C.byref(ds.layout), L.GM_F32, xs.data_ptr(), 8, L.GM_MAX, out.data_ptr(), None,
                                     None, 0, comm.comm, None, None))
