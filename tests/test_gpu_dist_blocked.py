"""Exchange-overlapped multi-GPU aggregation on ONE B200 ("P virtual ranks",
SURVEY.md §8e single-GPU test mode): each virtual rank splits its destination
rows by source block (gm_csr_split_blocks), runs the own-shard block, then
continues the rows' accumulation block by block as the emulated chunked
all-gathers land (gm_spmm_accumulate). The exchange is a D2D copy of the
other virtual ranks' shard chunks, exactly what all_gather_into_tensor
delivers.

Bar: the block split is a bit-exact stable partition; max/min values and
argmax ids equal the single-pass oracle bit-for-bit; sum/mean within the
condition-aware fp32 tolerance |gpu - ref64| <= 1e-5 * sum|x| + 1e-6 (one
re-association per block boundary)."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from paper_2507_16991_b200.dist import BlockedSpmm, chunk_layout, partition_rows_by_nnz, source_blocks
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


def _graph(n, e, f, kind=1, seed=77, quantize=1):
    lib = L.lib()
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    lib.gm_synth_edges_host(kind, seed, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    x = np.zeros((n, f), np.float32)
    lib.gm_synth_features_host(seed, 0, n, f, quantize, L.GM_F32, x.ctypes.data)
    return src, dst, x


class _VirtualExchange:
    """all_gather_into_tensor over virtual ranks: chunk c of every shard."""

    def __init__(self, shards, cs):
        self.shards, self.cs = shards, cs

    def for_rank(self, r):
        def ag(out, inp):
            c = (inp.data_ptr() - self.shards[r].data_ptr()) // (self.shards[r].stride(0) * inp.element_size())
            c //= self.cs
            for q, sh in enumerate(self.shards):
                out[q * self.cs:(q + 1) * self.cs].copy_(sh[c * self.cs:(c + 1) * self.cs])
            return None
        return ag


def _setup(n, e, f, world, chunks, dtype=torch.float32):
    src, dst, x = _graph(n, e, f)
    g = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, n)
    csc = g.to_csc()
    rp = csc.rowptr.cpu().numpy()
    cuts = partition_rows_by_nnz(rp, world)
    s_rows, cs = chunk_layout(n, world, chunks)
    xt = torch.from_numpy(x).cuda().to(dtype)
    shards = []
    for q in range(world):
        sh = torch.zeros(chunks * cs, f, dtype=dtype, device="cuda")
        lo, hi = q * s_rows, min((q + 1) * s_rows, n)
        if hi > lo:
            sh[: hi - lo].copy_(xt[lo:hi])
        shards.append(sh)
    ex = _VirtualExchange(shards, cs)
    ranks = []
    for r in range(world):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        view = csc.row_slice(r0, r1, int(rp[r1] - rp[r0]))
        ranks.append((r0, r1, BlockedSpmm(view, n, r, world, chunks, allgather=ex.for_rank(r))))
    return src, dst, x, csc, rp, shards, ranks


@pytest.mark.parametrize("world,chunks", [(1, 2), (2, 2), (3, 4), (4, 1)])
def test_split_blocks_is_stable_partition(world, chunks):
    n, e, f = 6000, 240000, 4
    src, dst, x, csc, rp, shards, ranks = _setup(n, e, f, world, chunks)
    col = csc.col.cpu().numpy()
    perm = csc.perm.cpu().numpy()
    for r, (r0, r1, bs) in enumerate(ranks):
        blk, cmap = (t.cpu().numpy() for t in source_blocks(n, r, world, chunks))
        nb = chunks + 1
        rpb = bs.rowptr_b.view(nb, -1).cpu().numpy()
        colb = bs.col_b.cpu().numpy()
        permb = bs.perm_b.cpu().numpy()
        tot = 0
        for b in range(nb):
            tot += rpb[b, -1] - rpb[b, 0]
        assert tot == rp[r1] - rp[r0]
        for v in range(r0, r1, max(1, (r1 - r0) // 300)):
            ks = np.arange(rp[v], rp[v + 1])
            for b in range(nb):
                sel = ks[blk[col[ks]] == b]
                a, z = rpb[b, v - r0], rpb[b, v - r0 + 1]
                assert np.array_equal(permb[a:z], perm[sel]), (r, v, b)
                assert np.array_equal(colb[a:z], cmap[col[sel]]), (r, v, b)


@pytest.mark.parametrize("world,chunks", [(2, 2), (3, 4), (4, 2)])
@pytest.mark.parametrize("kind", ["max", "min"])
def test_blocked_max_argmax_bit_exact(world, chunks, kind):
    n, e, f = 20000, 1_200_000, 33   # power-law hubs stay > 1024 per block
    src, dst, x, csc, rp, shards, ranks = _setup(n, e, f, world, chunks)
    orc = Oracle()
    rpo, colo, permo = orc.build_compressed(dst, src, n)
    want, warg = orc.spmm_max(rpo, colo, permo, x, is_min=kind == "min")
    for i, (r0, r1, bs) in enumerate(ranks):
        out, arg = bs(shards[i], kind)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == want[r0:r1].tobytes(), (r0, r1)
        assert np.array_equal(arg.cpu().numpy().astype(np.int64), warg[r0:r1]), (r0, r1)


@pytest.mark.parametrize("world,chunks", [(2, 2), (3, 4), (8, 2)])
@pytest.mark.parametrize("kind", ["sum", "mean"])
@pytest.mark.parametrize("f", [8, 100])
def test_blocked_sum_mean_tolerance(world, chunks, kind, f):
    n, e = 20000, 1_200_000
    src, dst, x, csc, rp, shards, ranks = _setup(n, e, f, world, chunks)
    orc = Oracle()
    rpo, colo, permo = orc.build_compressed(dst, src, n)
    ref = orc.spmm(rpo, colo, permo, x.astype(np.float64), mean=kind == "mean")
    scale = orc.spmm(rpo, colo, permo, np.abs(x).astype(np.float64), mean=kind == "mean")
    for i, (r0, r1, bs) in enumerate(ranks):
        out = bs(shards[i], kind)
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.float64)
        err = np.abs(got - ref[r0:r1])
        assert np.all(err <= 1e-5 * scale[r0:r1] + 1e-6), (i, float(err.max()))


def test_blocked_f64_sum_and_repeat_calls():
    n, e, f = 8000, 300000, 16
    src, dst, x, csc, rp, shards, ranks = _setup(n, e, f, 2, 3, dtype=torch.float64)
    orc = Oracle()
    rpo, colo, permo = orc.build_compressed(dst, src, n)
    ref = orc.spmm(rpo, colo, permo, x.astype(np.float64))
    for i, (r0, r1, bs) in enumerate(ranks):
        a = bs(shards[i], "sum").clone()
        b = bs(shards[i], "sum")   # buffers reused: same answer
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        assert np.allclose(a.cpu().numpy(), ref[r0:r1], rtol=1e-12, atol=1e-12)


def test_blocked_bf16_max_is_exact():
    # bf16 max/min never rounds, so the overlap mode is bit-exact in any dtype
    # (bf16 sums carry fp32 rows: tests/test_gpu_dist_push.py)
    n, e, f = 2000, 20000, 8
    src, dst, x, csc, rp, shards, ranks = _setup(n, e, f, 2, 2, dtype=torch.bfloat16)
    orc = Oracle()
    rpo, colo, permo = orc.build_compressed(dst, src, n)
    xb = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    want, warg = orc.spmm_max(rpo, colo, permo, xb)
    for i, (r0, r1, bs) in enumerate(ranks):
        out, arg = bs(shards[i], "max")
        torch.cuda.synchronize()
        assert np.array_equal(out.float().cpu().numpy(), want[r0:r1])
        assert np.array_equal(arg.cpu().numpy().astype(np.int64), warg[r0:r1])


# ---------------------------------------------------------------------------
# halo-only exchange (HaloSpmm) over virtual ranks
# ---------------------------------------------------------------------------
from paper_2507_16991_b200.dist import HaloSpmm, halo_need  # noqa: E402


def _halo_setup(n, e, f, world, dtype=torch.float32):
    src, dst, x = _graph(n, e, f)
    g = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, n)
    csc = g.to_csc()
    rp = csc.rowptr.cpu().numpy()
    cuts = partition_rows_by_nnz(rp, world)
    s_rows = -(-n // world)
    xt = torch.from_numpy(x).cuda().to(dtype)
    shards = []
    for q in range(world):
        sh = torch.zeros(s_rows, f, dtype=dtype, device="cuda")
        lo, hi = q * s_rows, min((q + 1) * s_rows, n)
        sh[: hi - lo].copy_(xt[lo:hi])
        shards.append(sh)
    views, needs = [], []
    for r in range(world):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        v = csc.row_slice(r0, r1, int(rp[r1] - rp[r0]))
        views.append((r0, r1, v))
        needs.append(halo_need(v, n, r, world))
    ranks = []
    for r in range(world):
        send = [needs[q][r] for q in range(world)]  # what q needs from me

        def a2a(recv, sendbuf, rs, ss, r=r):
            # what all_to_all_single delivers: from each peer q its pack for me
            parts = [shards[q][needs[r][q].long()] for q in range(world)]
            recv.copy_(torch.cat(parts))
            return None
        r0, r1, v = views[r]
        ranks.append((r0, r1, HaloSpmm(v, n, r, world, needs[r], send, alltoall=a2a)))
    return src, dst, x, shards, needs, ranks


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind", ["max", "sum", "mean"])
def test_halo_exchange_matches_oracle(world, kind):
    n, e, f = 20000, 1_200_000, 33
    src, dst, x, shards, needs, ranks = _halo_setup(n, e, f, world)
    orc = Oracle()
    rpo, colo, permo = orc.build_compressed(dst, src, n)
    if kind == "max":
        want, warg = orc.spmm_max(rpo, colo, permo, x)
    else:
        ref = orc.spmm(rpo, colo, permo, x.astype(np.float64), mean=kind == "mean")
        scale = orc.spmm(rpo, colo, permo, np.abs(x).astype(np.float64), mean=kind == "mean")
    for i, (r0, r1, hs) in enumerate(ranks):
        # the halo is exactly the referenced remote rows
        s_rows = -(-n // world)
        refd = np.unique(src[(dst >= r0) & (dst < r1)])
        remote = refd[(refd < i * s_rows) | (refd >= (i + 1) * s_rows)]
        assert hs.halo_rows() == remote.size
        res = hs(shards[i], kind)
        torch.cuda.synchronize()
        if kind == "max":
            out, arg = res
            assert out.cpu().numpy().tobytes() == want[r0:r1].tobytes()
            assert np.array_equal(arg.cpu().numpy().astype(np.int64), warg[r0:r1])
        else:
            err = np.abs(res.cpu().numpy().astype(np.float64) - ref[r0:r1])
            assert np.all(err <= 1e-5 * scale[r0:r1] + 1e-6), float(err.max())


def test_gather_rows_pack():
    lib = L.lib()
    for dtype, code, f in ((torch.float32, L.GM_F32, 33), (torch.bfloat16, L.GM_BF16, 128), (torch.float64, L.GM_F64, 5)):
        x = torch.randn(5000, f, device="cuda").to(dtype)
        idx = torch.randint(0, 5000, (3001,), device="cuda", dtype=torch.int32)
        out = torch.empty(3001, f, dtype=dtype, device="cuda")
        L.check(lib.gm_gather_rows(code, x.data_ptr(), f, idx.data_ptr(), 3001, out.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert torch.equal(out, x[idx.long()])
