"""segment_matmul (tcgen05 grouped GEMM) parity on B200.

Tolerance (stated, bf16 path — SURVEY.md §7.2/§8c): inputs are bf16 (rounded
on both sides), products are exact in fp32 and accumulate in fp32, so against
the fp64 oracle on the same rounded inputs
    |gpu - ref64| <= 1e-5 * sum_k |a_ik b_kj| + 1e-7             (fp32 output)
    |gpu - ref64| <= 2^-8 * |ref64| + 1e-5 * sum_k |a_ik b_kj|    (bf16 output)
"""
import os

import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ref_rows(x, ptr, w, rows):
    """fp64 reference and |a||b| scale for selected output rows."""
    x64 = x.double().cpu().numpy()
    w64 = w.double().cpu().numpy()
    ptr = np.asarray(ptr)
    g = np.searchsorted(ptr, rows, side="right") - 1
    ref = np.einsum("rk,rkn->rn", x64[rows], w64[g])
    scale = np.einsum("rk,rkn->rn", np.abs(x64[rows]), np.abs(w64[g]))
    return ref, scale


def check(out, x, ptr, w, rows, bf16_out):
    ref, scale = ref_rows(x, ptr, w, rows)
    got = out.double().cpu().numpy()[rows]
    err = np.abs(got - ref)
    tol = 1e-5 * scale + (2.0 ** -8 * np.abs(ref) if bf16_out else 1e-7)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} elements out of tolerance, max err {err.max():.3e}"


def test_golden_ragged_groups_fp32_and_bf16():
    d = np.load(os.path.join(GOLD, "gemm.npz"))
    x = torch.from_numpy(d["seg_x"]).cuda().to(torch.bfloat16)  # already bf16-exact
    w = torch.from_numpy(d["seg_w"]).cuda().to(torch.bfloat16)
    ptr = [int(v) for v in d["seg_ptr"]]
    ref = d["seg_out64"]  # the reference's grouped_matmul<double> on the rounded inputs
    scale = Oracle().segment_matmul(np.abs(d["seg_x"].astype(np.float64)), d["seg_ptr"],
                                    np.abs(d["seg_w"].astype(np.float64)))
    for dt in (torch.float32, torch.bfloat16):
        out = gm.segment_matmul(x, ptr, w, out_dtype=dt).double().cpu().numpy()
        tol = 1e-5 * scale + (2.0 ** -8 * np.abs(ref) if dt == torch.bfloat16 else 1e-7)
        assert np.all(np.abs(out - ref) <= tol), dt


@pytest.mark.parametrize("k,n", [(64, 16), (128, 128), (128, 48), (192, 256), (256, 64), (512, 512), (1024, 256)])
def test_shapes_and_ragged_tiles(k, n):
    torch.manual_seed(k * 1000 + n)
    ptr = [0, 5, 5, 133, 400, 401, 1031]
    x = torch.randn(ptr[-1], k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(len(ptr) - 1, k, n, device="cuda") / k ** 0.5).to(torch.bfloat16)
    for dt in (torch.float32, torch.bfloat16):
        out = gm.segment_matmul(x, ptr, w, out_dtype=dt)
        check(out, x, ptr, w, np.arange(ptr[-1]), dt == torch.bfloat16)


def test_ogb_mag_shape_sampled_rows():
    ptr = [0, 736_389, 1_871_038, 1_879_778, 1_939_743]
    torch.manual_seed(3)
    x = torch.randn(ptr[-1], 128, device="cuda").to(torch.bfloat16)
    w = (0.1 * torch.randn(4, 128, 128, device="cuda")).to(torch.bfloat16)
    out = gm.segment_matmul(x, ptr, w)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([rng.integers(0, ptr[-1], 4000), np.array(ptr[1:-1]) - 1,
                                     np.array(ptr[:-1]), [ptr[-1] - 1]]))
    check(out, x, ptr, w, rows, True)


def test_list_form_and_errors():
    torch.manual_seed(1)
    w = torch.randn(3, 64, 32, device="cuda").to(torch.bfloat16)
    hs = [torch.randn(r, 64, device="cuda").to(torch.bfloat16) for r in (1, 7, 3)]
    outs = gm.grouped_matmul(hs, w, out_dtype=torch.float32)
    assert [o.shape[0] for o in outs] == [1, 7, 3]
    for h, o, g in zip(hs, outs, range(3)):
        want = h.double() @ w[g].double()
        assert torch.allclose(o.double(), want, rtol=1e-5, atol=1e-5)
    # empty group -> 0 x F' (test_hetero.cpp:82-92)
    outs = gm.grouped_matmul([hs[0][:0], hs[1], hs[2]], w)
    assert outs[0].shape == (0, 32)
    with pytest.raises(ValueError, match="group count mismatch"):
        gm.grouped_matmul(hs[:2], w)
    with pytest.raises(ValueError, match="inner dimension mismatch"):
        gm.grouped_matmul([hs[0], hs[1], torch.zeros(2, 5, device="cuda")], w)



def test_odd_shapes_pad_internally():
    # the reference's own test shapes (test_hetero.cpp:61-106): K=3, N=5 / 4 / 2
    d = np.load(os.path.join(GOLD, "gemm.npz"))
    for xk, wk, ptr, ok in (("gm_x", "gm_w", [0, 2, 6], "gm_out"), ("gm_empty_x", "gm_empty_w", [0, 0, 2], "gm_empty_out")):
        x = torch.from_numpy(d[xk]).cuda().to(torch.bfloat16)
        w = torch.from_numpy(d[wk]).cuda().to(torch.bfloat16)
        got = gm.segment_matmul(x, ptr, w, out_dtype=torch.float32).double().cpu().numpy()
        # reference output on the bf16-rounded inputs
        want = Oracle().segment_matmul(x.double().cpu().numpy(), np.array(ptr), w.double().cpu().numpy())
        assert np.allclose(got, want, rtol=1e-6, atol=1e-6)
        # and within bf16 input rounding of the reference's f64 result
        assert np.allclose(got, d[ok], rtol=2e-2, atol=2e-2)
    for k, n in ((3, 5), (100, 7), (130, 33)):
        torch.manual_seed(k + n)
        ptr = [0, 17, 17, 300]
        x = torch.randn(ptr[-1], k, device="cuda").to(torch.bfloat16)
        w = torch.randn(3, k, n, device="cuda").to(torch.bfloat16)
        check(gm.segment_matmul(x, ptr, w, out_dtype=torch.float32), x, ptr, w, np.arange(ptr[-1]), False)


# ---------------------------------------------------------------------------
# fp32 operands: split-bf16 GEMM on the same tcgen05 kernel (gm_segment_matmul_f32)
# bar (north_star, fp32 GEMM): |gpu - ref64| <= 1e-5 * sum_k |x_ik||W_kj| + 1e-7
# ---------------------------------------------------------------------------
# k % 4 == 0: fused split (TMA fp32 tiles -> pieces in smem); otherwise the staged pieces path
@pytest.mark.parametrize("k,n", [(3, 5), (36, 40), (64, 16), (100, 7), (128, 128), (128, 512), (130, 33), (256, 64),
                                 (512, 256), (1024, 64)])
@pytest.mark.parametrize("ptr", [[0, 5, 5, 133, 400, 401, 1031], [0, 9000, 9001, 23000]])
def test_fp32_operands_meet_fp32_bound(k, n, ptr):
    torch.manual_seed(k * 7 + n)
    x = torch.randn(ptr[-1], k, device="cuda") * 3.0
    w = torch.randn(len(ptr) - 1, k, n, device="cuda") / k ** 0.5
    out = gm.segment_matmul(x, ptr, w)
    assert out.dtype == torch.float32
    ref = Oracle().segment_matmul(x.double().cpu().numpy(), np.array(ptr), w.double().cpu().numpy())
    scale = Oracle().segment_matmul(np.abs(x.double().cpu().numpy()), np.array(ptr), np.abs(w.double().cpu().numpy()))
    err = np.abs(out.double().cpu().numpy() - ref)
    assert np.all(err <= 1e-5 * scale + 1e-7), f"max err {err.max():.3e}, max rel-to-scale {(err / scale).max():.3e}"


def test_fp32_reference_golden_cases():
    # test_hetero.cpp:61-106 shapes (K=3 -> N=5/4/2), the reference's f64 outputs
    d = np.load(os.path.join(GOLD, "gemm.npz"))
    for xk, wk, ptr, ok in (("gm_x", "gm_w", [0, 2, 6], "gm_out"), ("gm_empty_x", "gm_empty_w", [0, 0, 2], "gm_empty_out")):
        x = torch.from_numpy(d[xk]).cuda().float()
        w = torch.from_numpy(d[wk]).cuda().float()
        got = gm.segment_matmul(x, ptr, w).double().cpu().numpy()
        scale = Oracle().segment_matmul(np.abs(d[xk].astype(np.float64)), np.array(ptr), np.abs(d[wk].astype(np.float64)))
        assert np.all(np.abs(got - d[ok]) <= 1e-5 * scale + 1e-7)
    outs = gm.grouped_matmul([torch.from_numpy(d["gm_x"][:2]).cuda().float(), torch.from_numpy(d["gm_x"][2:]).cuda().float()],
                             torch.from_numpy(d["gm_w"]).cuda().float())
    assert outs[0].dtype == torch.float32 and outs[1].shape[0] == 4


def test_packed_weights_cached_and_invalidated_by_inplace_update():
    torch.manual_seed(5)
    ptr = [0, 300, 300, 1000]
    x = torch.randn(ptr[-1], 128, device="cuda").to(torch.bfloat16)
    w = (torch.randn(3, 128, 64, device="cuda") / 11).to(torch.bfloat16)
    a = gm.segment_matmul(x, ptr, w, out_dtype=torch.float32)
    packed = w._gm_packed[2]
    b = gm.segment_matmul(x, ptr, w, out_dtype=torch.float32)
    assert w._gm_packed[2] is packed and torch.equal(a, b)  # reused, same result
    w.mul_(2)  # in-place update -> version bump -> re-pack
    c = gm.segment_matmul(x, ptr, w, out_dtype=torch.float32)
    assert w._gm_packed[2] is not packed
    check(c, x, ptr, w, np.arange(ptr[-1]), False)


# fp32 activations x bf16 weights (the hetero layer's bf16-W route): x is read
# as fp32 and rounded to bf16 inside the GEMM kernel (gm_segment_matmul_packed_xf32);
# the operands are exactly those of casting x first, so the result must match
# the cast-then-GEMM route bit for bit.
@pytest.mark.parametrize("k,n", [(128, 128), (36, 40), (100, 7), (256, 512)])
def test_fp32_activations_bf16_weights_match_cast_route(k, n):
    torch.manual_seed(k + n)
    ptr = [0, 5, 5, 133, 400, 401, 9031]
    x = torch.randn(ptr[-1], k, device="cuda") * 2.0
    w = (torch.randn(len(ptr) - 1, k, n, device="cuda") / k ** 0.5).to(torch.bfloat16)
    got = gm.segment_matmul(x, ptr, w, out_dtype=torch.float32)
    want = gm.segment_matmul(x.to(torch.bfloat16), ptr, w, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert got.dtype == torch.float32
    assert torch.equal(got, want), float((got - want).abs().max())


# ---------------------------------------------------------------------------
# grouped_matmul over separate tensors (hetero.hpp:134-157) through the
# pointer-array entry gm_grouped_matmul: per-group TMA maps, outputs written
# in place; the gathered fallback for shapes that need padding
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("k,n,groups", [(128, 128, 4), (64, 48, 3), (128, 256, 8), (100, 32, 3), (36, 40, 9)])
@pytest.mark.parametrize("route", ["f32", "f32x_bf16w", "bf16"])
def test_grouped_matmul_pointer_array(k, n, groups, route):
    torch.manual_seed(k + n + groups)
    rows = [0 if g == 1 else 300 * g + 7 for g in range(groups)]
    xs = [torch.randn(r, k, device="cuda") for r in rows]
    w = torch.randn(groups, k, n, device="cuda") / k ** 0.5
    if route == "f32x_bf16w":
        w = w.to(torch.bfloat16)
    if route == "bf16":
        xs = [x.to(torch.bfloat16) for x in xs]
        w = w.to(torch.bfloat16)
    odt = torch.float32
    outs = [torch.full((r, n), float("nan"), device="cuda") for r in rows]
    got = gm.grouped_matmul(xs, w, out_dtype=odt, out=outs)
    torch.cuda.synchronize()
    for g in range(groups):
        assert got[g].data_ptr() == outs[g].data_ptr()  # written in place
        xg = xs[g].double().cpu().numpy()
        if route != "f32":  # the bf16 operands the kernel multiplies
            xg = xs[g].to(torch.bfloat16).double().cpu().numpy()
        wg = w[g].double().cpu().numpy()
        ref = xg @ wg
        scale = np.abs(xg) @ np.abs(wg)
        assert np.all(np.abs(got[g].double().cpu().numpy() - ref) <= 1e-5 * scale + 1e-6), (route, g)


def test_grouped_matmul_matches_segment_matmul_bitwise():
    torch.manual_seed(9)
    rows = [700, 1, 0, 1234]
    xs = [torch.randn(r, 128, device="cuda") for r in rows]
    w = torch.randn(4, 128, 128, device="cuda") / 11
    got = gm.grouped_matmul(xs, w)
    ptr = np.concatenate([[0], np.cumsum(rows)]).tolist()
    want = gm.segment_matmul(torch.cat(xs), ptr, w)
    torch.cuda.synchronize()
    for g in range(4):
        assert torch.equal(got[g], want[ptr[g]:ptr[g + 1]])
