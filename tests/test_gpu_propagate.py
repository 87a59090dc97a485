"""Generic message passing on B200: select_path and propagate
(message_passing.hpp:14-36, 176-258), restating the reference's path tests
(test_message_passing.cpp:47-65 select_path rules, :150-176 paths agree,
:178-186 fused path rejects callbacks), plus a reference-produced check
(propagate with an edge-attribute message == the reference's weighted spmm,
bit for bit) and the undirected max/min grouping."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from oracle.oracle import Oracle, Reference

pytestmark = pytest.mark.gpu


def T(a):
    return torch.as_tensor(np.asarray(a)).cuda()


def rand_graph(n, e, seed, kind=0):
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    L.lib().gm_synth_edges_host(kind, seed, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    return src, dst


def test_select_path_honors_metadata_and_callbacks():
    # test_message_passing.cpp:47-65
    s = gm.EdgeIndex(T([1, 0, 2]), T([0, 1, 2]), 3, 3, sort_order="by_dst")
    assert gm.select_path(s, False) == gm.SEGMENT_FUSED
    assert gm.select_path(s, True) == gm.EDGE_MATERIALIZE
    plain = gm.EdgeIndex(T([1, 0, 2]), T([0, 2, 1]), 3, 3)
    assert gm.select_path(plain, False) == gm.EDGE_MATERIALIZE
    plain.to_csc()
    assert gm.select_path(plain, False) == gm.SEGMENT_FUSED
    sym = gm.EdgeIndex(T([0, 1]), T([1, 0]), 2, 2, is_undirected=True)
    assert gm.select_path(sym, False) == gm.EDGE_MATERIALIZE
    sym.to_csr()
    assert gm.select_path(sym, False) == gm.SEGMENT_FUSED


@pytest.mark.parametrize("agg", ["sum", "mean", "max", "min"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_propagate_paths_agree_bitwise(agg, dtype):
    # test_message_passing.cpp:150-176 with elementwise message/update functions
    src, dst = rand_graph(500, 6000, 70, kind=1)
    e = gm.EdgeIndex(T(src), T(dst), 500, 500)
    g = torch.Generator(device="cuda").manual_seed(1)
    h = (torch.floor((torch.rand(500, 7, device="cuda", generator=g) * 2 - 1) * 8) / 8).to(dtype)
    ea = torch.rand(6000, 1, device="cuda", generator=g).to(dtype)
    fns = gm.MessageFns(message=lambda hw, a, hv: hw * a - hv, update=lambda hv, a: hv + a)
    out_edge = gm.propagate(e, h, h, ea, fns, agg, gm.EDGE_MATERIALIZE)
    out_fused = gm.propagate(e, h, h, ea, fns, agg, gm.SEGMENT_FUSED)
    torch.cuda.synchronize()
    assert torch.equal(out_edge, out_fused)
    # identity message, no attribute: the fused path is the one-kernel SpMM
    ident = gm.MessageFns()
    a = gm.propagate(e, h, h, None, ident, agg, gm.EDGE_MATERIALIZE)
    b = gm.propagate(e, h, h, None, ident, agg, gm.SEGMENT_FUSED)
    assert torch.equal(a, b)
    assert torch.equal(b, gm.neighbor_aggregate(e, h, agg))


def test_propagate_edge_attribute_message_equals_reference_weighted_spmm():
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    src, dst = rand_graph(300, 3000, 5)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (300, 9)).astype(np.float32)
    w = rng.uniform(0.5, 1.5, 3000).astype(np.float32)
    e = gm.EdgeIndex(T(src), T(dst), 300, 300)
    fns = gm.MessageFns(message=lambda hw, a, hv: hw * a)
    xt = T(x)
    for path in (gm.EDGE_MATERIALIZE, gm.SEGMENT_FUSED):
        got = gm.propagate(e, xt, xt, T(w).reshape(-1, 1), fns, "sum", path).cpu().numpy()
        want = Reference().spmm(src, dst, 300, 300, x, w)
        assert got.tobytes() == want.tobytes(), path


def test_propagate_rejects_callback_on_fused_path_and_applies_it_on_edges():
    # test_message_passing.cpp:178-186
    e = gm.EdgeIndex(T([0]), T([1]), 2, 2)
    h = torch.rand(2, 2, device="cuda", dtype=torch.float64)
    with pytest.raises(ValueError):
        gm.propagate(e, h, h, None, gm.MessageFns(), "sum", gm.SEGMENT_FUSED, callback=lambda m, t: m)
    out = gm.propagate(e, h, h, None, gm.MessageFns(), "sum", gm.EDGE_MATERIALIZE, callback=lambda m, t: m * 3)
    assert torch.equal(out[1], h[0] * 3) and torch.equal(out[0], torch.zeros_like(out[0]))
    with pytest.raises(ValueError):
        gm.propagate(e, h[:1], h, None, gm.MessageFns(), "sum", gm.EDGE_MATERIALIZE)


def test_undirected_max_gathers_the_in_neighbour_and_names_the_forward_edge():
    src, dst = rand_graph(400, 3000, 9)
    s2, d2 = np.concatenate([src, dst]), np.concatenate([dst, src])  # symmetric multiset
    e = gm.EdgeIndex(T(s2), T(d2), 400, 400, is_undirected=True)
    rng = np.random.default_rng(2)
    x = (np.floor(rng.uniform(-1, 1, (400, 5)) * 8) / 8).astype(np.float32)
    out, arg = gm.neighbor_aggregate(e, T(x), "max", return_argmax=True)
    orc = Oracle()
    rp, col, perm = orc.build_compressed(d2, s2, 400)
    want, warg = orc.spmm_max(rp, col, perm, x)
    assert out.cpu().numpy().tobytes() == want.tobytes()
    assert np.array_equal(arg.cpu().numpy().astype(np.int64), warg)
    edge = gm.propagate(e, T(x), T(x), None, gm.MessageFns(), "max", gm.EDGE_MATERIALIZE)
    assert torch.equal(edge, out)


def test_gather_rows_bounds_error_shape():
    x = torch.rand(3, 2, device="cuda")
    with pytest.raises(IndexError, match="index 5 at position 1 outside"):
        gm.gather_rows(x, torch.tensor([0, 5], device="cuda"))
