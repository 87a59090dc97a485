"""Push mode (the exchange of the next layer fused into this layer's SpMM
epilogue, gm_spmm_ex push) and the bf16 fp32-carry of the overlap modes, on
ONE B200 with P virtual ranks (SURVEY.md §8e single-GPU test mode): every
virtual rank owns an [N, F] replica of the layer input; its SpMM over its
destination rows stores each finished row into its own next-layer replica and
into the other ranks' replicas (plain device pointers here; CUDA IPC mappings
over NVLink across GPUs).

Bar: push mode is bit-identical to the single-GPU gm_spmm for every row a
replica needs (full push: all rows; halo masks: the rows that rank
references), over two ping-pong layers; bf16 blocked/halo sums with the fp32
carry meet |gpu - ref64| <= 1e-5 * sum|x| + 2^-8 |ref| (one rounding per row)."""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from paper_2507_16991_b200.dist import (BlockedSpmm, HaloSpmm, PushSpmm, chunk_layout, halo_need,
                                        partition_rows_by_nnz, push_masks)
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


def _graph(n, e, f, dtype, seed=91):
    lib = L.lib()
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    lib.gm_synth_edges_host(1, seed, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    x = np.zeros((n, f), np.float32)
    lib.gm_synth_features_host(seed, 0, n, f, 1, L.GM_F32, x.ctypes.data)
    g = gm.EdgeIndex(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, n)
    return src, dst, g, torch.from_numpy(x).cuda().to(dtype)


def _ranks(g, n, world):
    csc = g.to_csc()
    rp = csc.rowptr.cpu().numpy()
    cuts = partition_rows_by_nnz(rp, world)
    out = []
    for r in range(world):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        out.append((r0, r1, csc.row_slice(r0, r1, int(rp[r1] - rp[r0]))))
    return out


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("dtype,f,reduce", [(torch.float32, 100, "sum"), (torch.float32, 33, "mean"),
                                             (torch.bfloat16, 128, "sum"), (torch.bfloat16, 64, "mean"),
                                             (torch.float32, 8, "sum"), (torch.float32, 602, "mean"),
                                             (torch.float32, 100, "max"), (torch.bfloat16, 128, "min")])
@pytest.mark.parametrize("halo", [False, True])
def test_push_two_layers_bit_identical(world, dtype, f, reduce, halo):
    n, e = 20000, 900_000   # power-law: hub rows take the hub kernel's push path too
    src, dst, g, x = _graph(n, e, f, dtype)
    ranks = _ranks(g, n, world)
    bitmaps = []
    for r0, r1, v in ranks:
        mark = torch.empty(n, dtype=torch.uint8, device="cuda")
        cs = v.c_struct()
        L.check(L.lib().gm_mark_columns(C_byref(cs), mark.data_ptr(), torch.cuda.current_stream().cuda_stream))
        bitmaps.append(mark)
    allm = torch.stack(bitmaps)
    masks = [push_masks(v, n, r0, r1, r, world, gather=lambda m: allm) if halo else None
             for r, (r0, r1, v) in enumerate(ranks)]
    A = [x.clone() for _ in range(world)]
    B = [torch.full_like(x, float("nan")) for _ in range(world)]
    ops = [PushSpmm(v, r0, r1, r, world, masks[r]) for r, (r0, r1, v) in enumerate(ranks)]
    maxmin = reduce in ("max", "min")
    if maxmin:
        want1, warg1 = gm.neighbor_aggregate(g, x, reduce, return_argmax=True)
        want2, warg2 = gm.neighbor_aggregate(g, want1, reduce, return_argmax=True)
    else:
        want1 = gm.spmm(g, x, None, reduce)
        want2 = gm.spmm(g, want1, None, reduce)
        warg1 = warg2 = None
    for src_bufs, dst_bufs, want, warg in ((A, B, want1, warg1), (B, A, want2, warg2)):
        for r in range(world):
            res = ops[r](src_bufs[r], dst_bufs[r], [t.data_ptr() for t in dst_bufs], reduce)
            if maxmin:
                r0, r1 = ranks[r][0], ranks[r][1]
                assert torch.equal(res[1], warg[r0:r1]), ("argmax", r)
        torch.cuda.synchronize()
        for q, (r0, r1, v) in enumerate(ranks):
            got = dst_bufs[q]
            assert torch.equal(got[r0:r1], want[r0:r1]), ("own rows", q)
            need = (allm[q] != 0) if halo else torch.ones(n, dtype=torch.bool, device="cuda")
            need[r0:r1] = True
            assert torch.equal(got[need], want[need]), ("needed rows", q)
        if halo:   # a halo replica is only complete where it is read; refill the rest for the next layer
            for q in range(world):
                dst_bufs[q].copy_(want)


def C_byref(s):
    import ctypes
    return ctypes.byref(s)


def test_push_validation():
    n, e, f = 2000, 20000, 8
    src, dst, g, x = _graph(n, e, f, torch.float32)
    (r0, r1, v), = _ranks(g, n, 1)
    ep = L.gm_spmm_epilogue()
    ep.n_push = L.GM_MAX_PUSH + 1
    cs = v.c_struct()
    out = torch.empty_like(x)
    st = L.lib().gm_spmm_ex(C_byref(cs), C_byref(v.plan(f * 4)), L.GM_F32, x.data_ptr(), f, None, L.GM_SUM, 0, None,
                            C_byref(ep), out.data_ptr(), None, None)
    assert st == L.GM_ERR_INVALID_ARGUMENT


def _bf16_ref(src, dst, x_bf16, n, reduce):
    orc = Oracle()
    xs = x_bf16.float().cpu().numpy().astype(np.float64)
    rpo, colo, permo = orc.build_compressed(dst, src, n)
    ref = orc.spmm(rpo, colo, permo, xs, mean=reduce == "mean")
    scale = orc.spmm(rpo, colo, permo, np.abs(xs), mean=reduce == "mean")
    return ref, scale


class _VirtualExchange:
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


@pytest.mark.parametrize("world,chunks", [(2, 2), (4, 3)])
@pytest.mark.parametrize("reduce", ["sum", "mean"])
@pytest.mark.parametrize("f", [128, 8])
def test_blocked_bf16_carry(world, chunks, reduce, f):
    n, e = 20000, 1_200_000
    src, dst, g, x = _graph(n, e, f, torch.bfloat16)
    s_rows, cs = chunk_layout(n, world, chunks)
    shards = []
    for q in range(world):
        sh = torch.zeros(chunks * cs, f, dtype=torch.bfloat16, device="cuda")
        lo, hi = q * s_rows, min((q + 1) * s_rows, n)
        sh[: hi - lo].copy_(x[lo:hi])
        shards.append(sh)
    ex = _VirtualExchange(shards, cs)
    ref, scale = _bf16_ref(src, dst, x, n, reduce)
    for r, (r0, r1, v) in enumerate(_ranks(g, n, world)):
        out = BlockedSpmm(v, n, r, world, chunks, allgather=ex.for_rank(r))(shards[r], reduce)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy().astype(np.float64)
        err = np.abs(got - ref[r0:r1])
        assert np.all(err <= 1e-5 * scale[r0:r1] + 2.0 ** -8 * np.abs(ref[r0:r1]) + 1e-30), (r, float(err.max()))


@pytest.mark.parametrize("reduce", ["sum", "mean"])
def test_halo_bf16_carry(reduce):
    n, e, f, world = 20000, 1_200_000, 128, 3
    src, dst, g, x = _graph(n, e, f, torch.bfloat16)
    s_rows = -(-n // world)
    shards = []
    for q in range(world):
        sh = torch.zeros(s_rows, f, dtype=torch.bfloat16, device="cuda")
        lo, hi = q * s_rows, min((q + 1) * s_rows, n)
        sh[: hi - lo].copy_(x[lo:hi])
        shards.append(sh)
    ref, scale = _bf16_ref(src, dst, x, n, reduce)
    ranks = _ranks(g, n, world)
    needs = [halo_need(v, n, r, world) for r, (r0, r1, v) in enumerate(ranks)]
    for r, (r0, r1, v) in enumerate(ranks):
        send = [needs[q][r] for q in range(world)]   # what every peer needs from my shard

        def a2a(out, inp, rs, ss, r=r):
            off = 0
            for q in range(world):
                rows = needs[r][q].long()
                out[off: off + rows.numel()].copy_(shards[q][rows])
                off += rows.numel()
            return None
        op = HaloSpmm(v, n, r, world, needs[r], send, alltoall=a2a)
        out = op(shards[r], reduce)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy().astype(np.float64)
        err = np.abs(got - ref[r0:r1])
        assert np.all(err <= 1e-5 * scale[r0:r1] + 2.0 ** -8 * np.abs(ref[r0:r1]) + 1e-30), (r, float(err.max()))
