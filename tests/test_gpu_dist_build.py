"""Distributed build_compressed (dist.build_local_csc phases) over P virtual
ranks on ONE B200: each rank holds one contiguous chunk of the COO list; the
degree all-reduce, nnz cuts, owner routing (a stable grouping by owner through
gm_build_compressed) and the local stable build must give every rank exactly
the single-GPU CSC's rows [r0, r1): rowptr (rebased), col and global perm
bit-identical (edge_index.cpp:45-62 is a stable counting sort)."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from paper_2507_16991_b200.dist import (cuts_from_degrees, local_csc_from_routed, local_degrees,
                                        partition_rows_by_nnz, route_edges)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("n,e,kind", [(50_000, 2_000_000, 1), (300_000, 1_000_000, 0), (1_000, 200_000, 1)])
def test_local_csc_equals_global_rows(world, n, e, kind):
    src = torch.empty(e, dtype=torch.int64, device="cuda")
    dst = torch.empty(e, dtype=torch.int64, device="cuda")
    L.check(L.lib().gm_synth_edges(kind, 17, 0, e, n, n, src.data_ptr(), dst.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
    g = gm.EdgeIndex(src, dst, n, n)
    csc = g.to_csc()
    rp = csc.rowptr.cpu().numpy()
    chunks = [(q * e // world, (q + 1) * e // world) for q in range(world)]
    deg = sum(local_degrees(dst[a:b], n) for a, b in chunks)
    cuts = cuts_from_degrees(deg, world)
    assert np.array_equal(cuts, partition_rows_by_nnz(rp, world))
    routed = [route_edges(src[a:b], dst[a:b], a, cuts) for a, b in chunks]
    offs = [np.concatenate([[0], np.cumsum(r[3])]) for r in routed]
    for r in range(world):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        parts = [[routed[q][i][offs[q][r]:offs[q][r + 1]] for q in range(world)] for i in range(3)]
        s, d, eid = (torch.cat(p) for p in parts)
        loc = local_csc_from_routed(s, d, eid, r0, r1, n)
        assert loc.num_entries() == rp[r1] - rp[r0]
        assert torch.equal(loc.rowptr, csc.rowptr[r0:r1 + 1] - csc.rowptr[r0]), r
        k0, k1 = int(rp[r0]), int(rp[r1])
        assert torch.equal(loc.col, csc.col[k0:k1]), r
        assert torch.equal(loc.perm, csc.perm[k0:k1]), r


def test_more_ranks_than_rows_and_empty_chunks():
    # 8 ranks over 5 rows and 7 edges: most ranks own no rows, some chunks are empty
    n, world = 5, 8
    src = torch.tensor([0, 4, 2, 2, 1, 3, 0], dtype=torch.int64, device="cuda")
    dst = torch.tensor([1, 1, 4, 0, 1, 3, 3], dtype=torch.int64, device="cuda")
    e = src.numel()
    csc = gm.EdgeIndex(src, dst, n, n).to_csc()
    rp = csc.rowptr.cpu().numpy()
    chunks = [(q * e // world, (q + 1) * e // world) for q in range(world)]
    deg = sum(local_degrees(dst[a:b], n) for a, b in chunks)
    cuts = cuts_from_degrees(deg, world)
    routed = [route_edges(src[a:b], dst[a:b], a, cuts) for a, b in chunks]
    offs = [np.concatenate([[0], np.cumsum(r[3])]) for r in routed]
    total = 0
    for r in range(world):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        parts = [[routed[q][i][offs[q][r]:offs[q][r + 1]] for q in range(world)] for i in range(3)]
        s, d, eid = (torch.cat(p) for p in parts)
        loc = local_csc_from_routed(s, d, eid, r0, r1, n)
        k0, k1 = int(rp[r0]), int(rp[r1])
        assert torch.equal(loc.rowptr, csc.rowptr[r0:r1 + 1] - csc.rowptr[r0])
        assert torch.equal(loc.col, csc.col[k0:k1]) and torch.equal(loc.perm, csc.perm[k0:k1])
        total += loc.num_entries()
    assert total == e
