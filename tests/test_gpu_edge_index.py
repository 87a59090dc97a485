"""GPU-side EdgeIndex lifecycle: sort_by with the
carried cache and the undirected multiset claim, restating the reference's
own tests (test_edge_index.cpp:45-53, 142-172) against the device path, plus
large seeded cases checked against numpy's stable sort (the reference
test's own oracle, std::stable_sort)."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
import refrng

pytestmark = pytest.mark.gpu


def H(t):
    return t.cpu().numpy()


def test_sort_by_reference_case():
    # test_edge_index.cpp:142-172
    e = gm.EdgeIndex([2, 0, 1], [0, 1, 2], 3, 3)
    s, perm = e.sort_by("by_src")
    assert H(s.src()).tolist() == [0, 1, 2]
    assert H(perm).tolist() == [1, 2, 0]
    assert s.sort_order() == "by_src"
    assert s.has_csr_cache()
    again, perm2 = s.sort_by("by_src")
    assert H(perm2).tolist() == [0, 1, 2]
    stream = refrng.test_stream(22)
    src = [stream.next_below(9) for _ in range(100)]
    dst = [stream.next_below(9) for _ in range(100)]
    big = gm.EdgeIndex(src, dst, 9, 9)
    bs, bp = big.sort_by("by_dst")
    ref = np.argsort(np.asarray(dst), kind="stable")
    assert np.array_equal(H(bp), ref)
    assert np.array_equal(H(bs.src()), np.asarray(src)[ref])
    assert np.array_equal(H(bs.dst()), np.asarray(dst)[ref])
    with pytest.raises(ValueError):
        e.sort_by("unsorted")


@pytest.mark.parametrize("order", ["by_src", "by_dst"])
def test_sort_by_large_and_carried_cache(order):
    n, e = 50_000, 2_000_000
    lib = L.lib()
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    lib.gm_synth_edges_host(1, 31, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    g = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, n)
    s, perm = g.sort_by(order)
    keys = src if order == "by_src" else dst
    ref = np.argsort(keys, kind="stable")
    assert np.array_equal(H(perm), ref)
    assert np.array_equal(H(s.src()), src[ref]) and np.array_equal(H(s.dst()), dst[ref])
    # the sort claim holds on the new arrays and the carried view equals a fresh build
    gm.EdgeIndex(s.src(), s.dst(), n, n, sort_order=order)
    carried = s.to_csr() if order == "by_src" else s.to_csc()
    fresh = gm.build_compressed(s.src() if order == "by_src" else s.dst(),
                                s.dst() if order == "by_src" else s.src(), n, n)
    assert torch.equal(carried.rowptr, fresh.rowptr)
    assert torch.equal(carried.col, fresh.col)
    assert torch.equal(carried.perm, fresh.perm)  # identity
    assert (s.csr_build_count() if order == "by_src" else s.csc_build_count()) == 0


def test_undirected_claim_reference_cases():
    # test_edge_index.cpp:45-53
    assert gm.EdgeIndex([0, 1], [1, 0], 2, 2, is_undirected=True).is_undirected()
    with pytest.raises(ValueError, match="position 0 "):
        gm.EdgeIndex([0, 1], [1, 2], 3, 3, is_undirected=True)
    with pytest.raises(ValueError):
        gm.EdgeIndex([0, 0, 1], [1, 1, 0], 2, 2, is_undirected=True)
    assert gm.EdgeIndex([0, 0, 1, 1], [1, 1, 0, 0], 2, 2, is_undirected=True).is_undirected()


def test_undirected_claim_large_first_violation():
    rng = np.random.default_rng(5)
    n, half = 100_000, 1_500_000
    u = rng.integers(0, n, half)
    v = rng.integers(0, n, half)
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    p = rng.permutation(src.size)
    src, dst = src[p], dst[p]
    g = gm.EdgeIndex(src, dst, n, n, is_undirected=True)
    assert g.is_undirected()
    # break one reverse edge: the first position whose multiplicity differs
    bad = src.size // 3
    dst2 = dst.copy()
    dst2[bad] = (dst2[bad] + 1) % n
    fwd = {}
    for a, b in zip(src.tolist(), dst2.tolist()):
        fwd[(a, b)] = fwd.get((a, b), 0) + 1
    want = next(i for i, (a, b) in enumerate(zip(src.tolist(), dst2.tolist())) if fwd.get((b, a), 0) != fwd[(a, b)])
    with pytest.raises(ValueError, match=f"position {want} "):
        gm.EdgeIndex(src, dst2, n, n, is_undirected=True)
