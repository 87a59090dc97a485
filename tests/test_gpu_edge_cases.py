"""Degenerate shapes through the public API on B200 (the reference's own
edge-case tests: empty edge sets, empty groups, isolated rows — test_edge_index
.cpp:79-84, test_aggregate.cpp:35-46, test_hetero.cpp:61-92): no launch may
fault, every output keeps the reference's values (zeros / -1 argmax for empty
rows, 0 x F' blocks for empty groups)."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _empty_graph(n_src, n_dst):
    z = torch.empty(0, dtype=torch.int64, device="cuda")
    return gm.EdgeIndex(z, z, n_src, n_dst)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
@pytest.mark.parametrize("f", [1, 3, 100])
def test_empty_edge_set(dtype, f):
    g = _empty_graph(7, 5)
    x = torch.randn(7, f, device="cuda").to(dtype)
    for red in ("sum", "mean"):
        out = gm.spmm(g, x, None, red)
        torch.cuda.synchronize()
        assert out.shape == (5, f) and not out.float().abs().any()
    mx, arg = gm.neighbor_aggregate(g, x, "max", return_argmax=True)
    torch.cuda.synchronize()
    assert not mx.float().abs().any() and bool((arg == -1).all())
    csc = g.to_csc()
    assert csc.rowptr.cpu().tolist() == [0] * 6


def test_isolated_rows_and_single_edge():
    # rows 0, 2, 4 have no in-edges; one edge 3 -> 1
    g = gm.EdgeIndex(torch.tensor([3], device="cuda"), torch.tensor([1], device="cuda"), 5, 5)
    x = torch.arange(5 * 4, dtype=torch.float32, device="cuda").view(5, 4)
    out = gm.spmm(g, x, None, "mean")
    want = torch.zeros(5, 4, device="cuda")
    want[1] = x[3]
    assert torch.equal(out, want)
    mx, arg = gm.neighbor_aggregate(g, x, "max", return_argmax=True)
    assert torch.equal(mx, want)
    assert arg[1].tolist() == [0, 0, 0, 0] and bool((arg[[0, 2, 3, 4]] == -1).all())
    dx = gm.neighbor_aggregate_backward(g, "max", torch.ones(5, 4, device="cuda"), arg)
    wdx = torch.zeros(5, 4, device="cuda")
    wdx[3] = 1
    assert torch.equal(dx, wdx)


def test_backward_on_empty_graph():
    g = _empty_graph(6, 4)
    x = torch.randn(6, 8, device="cuda")
    w = torch.empty(0, device="cuda")
    dx, dw = gm.spmm_backward(g, x, w, "sum", torch.randn(4, 8, device="cuda"))
    torch.cuda.synchronize()
    assert dx.shape == (6, 8) and not dx.abs().any() and dw.numel() == 0


@pytest.mark.parametrize("fp32", [False, True])
def test_segment_matmul_empty_groups(fp32):
    ptr = [0, 0, 130, 130, 131]
    x = torch.randn(131, 64, device="cuda")
    w = torch.randn(4, 64, 32, device="cuda") / 8
    if not fp32:
        x, w = x.bfloat16(), w.bfloat16()
    y = gm.segment_matmul(x, ptr, w, out_dtype=torch.float32)
    ref = torch.cat([x[ptr[g]:ptr[g + 1]].double() @ w[g].double() for g in range(4)])
    assert y.shape == (131, 32)
    tol = 1e-5 * (x.double().abs() @ w[0].double().abs()).max().item() * 4 + 1e-6
    assert (y.double() - ref).abs().max().item() <= max(tol, 1e-2 if not fp32 else tol)


def test_build_compressed_single_row_and_all_in_one_row():
    keys = torch.zeros(5000, dtype=torch.int64, device="cuda")
    vals = torch.arange(5000, dtype=torch.int64, device="cuda").flip(0)
    v = gm.build_compressed(keys, vals, 1)
    rp, col, perm = v.to_host()
    assert rp.tolist() == [0, 5000]
    assert np.array_equal(perm.numpy(), np.arange(5000))          # stable: COO order kept
    assert np.array_equal(col.numpy(), np.arange(5000)[::-1])


@pytest.mark.parametrize("slice_kernel", ["1", "0"])
def test_edge_dot_on_a_row_slice(slice_kernel, monkeypatch):
    """gm_edge_dot_csc over a CSC row slice (rowptr[0] != 0, as a multi-GPU rank
    holds it) writes exactly the slice's entries, equal to the full call's."""
    import ctypes as C
    import subprocess
    import sys
    code = f"""
import ctypes as C, torch, numpy as np, sys
sys.path.insert(0, {repr(str(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))})
import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
n, e, f = 3000, 90000, 20
s = torch.empty(e, dtype=torch.int64, device='cuda'); d = torch.empty_like(s)
L.check(L.lib().gm_synth_edges(1, 5, 0, e, n, n, s.data_ptr(), d.data_ptr(), None))
g = gm.EdgeIndex(s, d, n, n); csc = g.to_csc()
x = torch.randn(n, f, device='cuda'); go = torch.randn(n, f, device='cuda')
def run(view, rows, a):  # a: the gradient rows of the view's destinations (local row ids)
    out = torch.full((e,), float('nan'), device='cuda')
    cs = view.c_struct()
    L.check(L.lib().gm_edge_dot_csc(L.GM_F32, C.byref(cs), C.byref(csc.plan()), rows.data_ptr(), a.data_ptr(), x.data_ptr(), f, out.data_ptr(), None))
    torch.cuda.synchronize(); return out
full = run(csc, csc.entry_rows(), go)
rp = csc.rowptr.cpu().numpy(); r0, r1 = 1000, 2200
view = csc.row_slice(r0, r1, int(rp[r1] - rp[r0]))
part = run(view, view.entry_rows(), go[r0:])
sel = csc.perm[int(rp[r0]):int(rp[r1])].long()
assert torch.equal(part[sel], full[sel])
mask = torch.ones(e, dtype=torch.bool, device='cuda'); mask[sel] = False
assert bool(torch.isnan(part[mask]).all())
print('ok')
"""
    env = dict(__import__('os').environ, GM_EDGE_DOT_SLICE=slice_kernel)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_host_operands_rejected_on_a_device_index():
    """A host tensor beside a device index fails loudly (ValueError) instead of
    reaching a kernel as a host pointer."""
    src = torch.tensor([0, 1, 2], device="cuda")
    dst = torch.tensor([1, 2, 0], device="cuda")
    g = gm.EdgeIndex(src, dst, 3, 3)
    xh = torch.ones(3, 4)
    with pytest.raises(ValueError, match="must be on cuda"):
        gm.spmm(g, xh, None, "sum")
    with pytest.raises(ValueError, match="must be on cuda"):
        gm.neighbor_aggregate(g, xh, "max", return_argmax=True)
    xd = torch.ones(3, 4, device="cuda")
    with pytest.raises(ValueError, match="must be on cuda"):
        gm.spmm_backward(g, xd, None, "sum", torch.ones(3, 4))
    with pytest.raises(ValueError, match="must be on cuda"):
        gm.gcn_layer(g, xd, torch.ones(4, 4), torch.zeros(4, device="cuda"))


@pytest.mark.parametrize("reduce", ["sum", "max"])
def test_window_size_is_pure_scheduling(reduce):
    """gm_spmm_plan_build's window size (auto: 1024 entries halved to keep >= 8
    waves of warps; or caller-set) changes scheduling only: the same output bits
    (and argmax ids) for auto, 256 and 4096 entry windows."""
    import ctypes as C
    import bench
    n, e, f = 100_000, 20_000_000, 36
    stream = torch.cuda.current_stream().cuda_stream
    g, x = bench.make_graph(gm, L, n, e, f, "cuda", stream)
    csc = g.to_csc()
    cs = csc.c_struct()
    lib = L.lib()
    nbytes = lib.gm_spmm_plan_bytes(cs.num_rows, cs.num_cols, cs.nnz)
    outs = []
    for win in (0, 256, 4096):
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        plan = L.gm_spmm_plan()
        plan.window_edges = win
        L.check(lib.gm_spmm_plan_build(C.byref(cs), C.c_void_p(buf.data_ptr()), nbytes, C.byref(plan),
                                       C.c_void_p(stream)))
        # auto: (E + N) / 1024 = 19.6k windows < 8 waves (37,888 warps) -> 512
        assert plan.window_edges == {0: 512, 256: 256, 4096: 4096}[win]
        out = torch.empty(n, f, device="cuda")
        arg = torch.empty(n, f, dtype=torch.int32, device="cuda") if reduce == "max" else None
        L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), f, None, None,
                            L.GM_MAX if reduce == "max" else L.GM_SUM, C.c_void_p(out.data_ptr()),
                            C.c_void_p(arg.data_ptr()) if arg is not None else None, C.c_void_p(stream)))
        torch.cuda.synchronize()
        outs.append((out, arg))
    for out, arg in outs[1:]:
        assert torch.equal(out, outs[0][0])
        if reduce == "max":
            assert torch.equal(arg, outs[0][1])
