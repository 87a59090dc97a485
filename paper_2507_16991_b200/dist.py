"""Multi-GPU destination-row partitioning + source-feature exchange
(north_star / SURVEY.md §8e).

Each destination row depends only on its in-edges, so the path shards by
contiguous destination-row ranges with one real exchange per SpMM: the
source-feature all-gather. Ranks own equal row shards of X (padded), all-gather
them every step (NCCL over NVLink on B200; gloo in the CPU tests) and run the
SpMM kernel on their own CSC row slice. Per-row results are unchanged, so the
multi-GPU output is bit-identical to the single-GPU one.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L


def partition_rows_by_nnz(rowptr: np.ndarray, parts: int) -> np.ndarray:
    """gm_partition_rows_by_nnz: cuts[p] = first row with rowptr >= p*E/parts."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    cuts = np.zeros(parts + 1, np.int64)
    L.check(L.lib().gm_partition_rows_by_nnz(rowptr.ctypes.data_as(C.POINTER(C.c_int64)), rowptr.size - 1,
                                             parts, cuts.ctypes.data_as(C.POINTER(C.c_int64))), "partition")
    return cuts


@dataclass
class Shard:
    rank: int
    world: int
    row_begin: int   # this rank's destination rows [row_begin, row_end)
    row_end: int
    shard_rows: int  # equal X shard height (padded)

    def x_rows(self):
        return self.rank * self.shard_rows, (self.rank + 1) * self.shard_rows


def make_shard(rowptr: np.ndarray, num_src_rows: int, rank: int, world: int) -> Shard:
    cuts = partition_rows_by_nnz(rowptr, world)
    return Shard(rank, world, int(cuts[rank]), int(cuts[rank + 1]), -(-num_src_rows // world))


def allgather_features(x_shard: torch.Tensor, shard: Shard, group=None, out=None) -> torch.Tensor:
    """Exchange step: every rank receives every shard ([world*shard_rows, F])."""
    full = out if out is not None else torch.empty(
        (shard.shard_rows * shard.world,) + tuple(x_shard.shape[1:]), dtype=x_shard.dtype, device=x_shard.device)
    dist.all_gather_into_tensor(full, x_shard.contiguous(), group=group)
    return full


# ---------------------------------------------------------------------------
# Distributed build_compressed: every rank holds one contiguous chunk of the
# COO edge list (edges [first_eid, first_eid + len), e.g. its file shard) and
# ends with the CSC row slice of its destination rows — global source ids in
# col, global COO positions in perm — without any rank holding the whole graph:
#   1. in-degrees of the local chunk (gm_degree), summed over ranks;
#   2. nnz-balanced row cuts from the global degrees;
#   3. each edge routed to the rank owning its destination (a stable grouping
#      by owner = gm_build_compressed over owner ids), one all_to_all;
#   4. the received edges (from rank q: q's chunk, ascending COO position; in q
#      order: ascending overall) compressed locally, perm mapped back to the
#      global positions. Stable at every step, so the slice is bit-identical to
#      the single-GPU CSC's rows [r0, r1).
# The phases are separate functions so one process can drive virtual ranks.
# ---------------------------------------------------------------------------
def local_degrees(dst: torch.Tensor, num_nodes: int) -> torch.Tensor:
    from .graphmill import _p, _stream
    deg = torch.empty(num_nodes, dtype=torch.int32, device=dst.device)
    L.check(L.lib().gm_degree(_p(dst), dst.numel(), num_nodes, _p(deg), _stream()), "gm_degree")
    return deg


def cuts_from_degrees(deg: torch.Tensor, world: int) -> np.ndarray:
    rowptr = np.zeros(deg.numel() + 1, np.int64)
    np.cumsum(deg.cpu().numpy().astype(np.int64), out=rowptr[1:])
    return partition_rows_by_nnz(rowptr, world)


def route_edges(src: torch.Tensor, dst: torch.Tensor, first_eid: int, cuts: np.ndarray):
    """(src, dst, eid) of the local chunk grouped stably by owner rank, and the
    per-owner counts (host list)."""
    from .graphmill import build_compressed
    world = len(cuts) - 1
    dev = dst.device
    owner = torch.searchsorted(torch.from_numpy(np.ascontiguousarray(cuts[1:])).to(dev), dst, right=True)
    pos = torch.arange(dst.numel(), dtype=torch.int64, device=dev)
    grp = build_compressed(owner, pos, world)  # stable grouping: perm = positions in owner order
    order = grp.perm.to(torch.int64)
    counts = (grp.rowptr[1:] - grp.rowptr[:-1]).cpu().tolist()
    return src[order], dst[order], order + first_eid, counts


def local_csc_from_routed(src: torch.Tensor, dst: torch.Tensor, eid: torch.Tensor, r0: int, r1: int,
                          num_nodes: int):
    """CSC row slice of rows [r0, r1) from the edges routed to this rank (in
    ascending COO position): rowptr rebased to 0, global col / perm."""
    from .graphmill import CsrView, build_compressed
    loc = build_compressed(dst - r0, src, r1 - r0, num_nodes)
    perm = eid[loc.perm.to(torch.int64)].to(torch.int32)
    return CsrView(loc.rowptr, loc.col, perm, num_nodes, dst.numel())


def _alltoall_rows(tensors, send_counts, group=None):
    """all_to_all_single of several same-length int64 tensors with one split
    plan (gloo: through host memory)."""
    world = dist.get_world_size(group)
    dev = tensors[0].device
    cpu = dist.get_backend(group) == "gloo"
    sc = torch.tensor(send_counts, dtype=torch.int64, device="cpu" if cpu else dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = rc.cpu().tolist()
    outs = []
    for t in tensors:
        inp = t.cpu() if cpu else t
        out = torch.empty(sum(recv_counts), dtype=t.dtype, device=inp.device)
        dist.all_to_all_single(out, inp, output_split_sizes=recv_counts, input_split_sizes=list(send_counts),
                               group=group)
        outs.append(out.to(dev))
    return outs


def build_local_csc(src: torch.Tensor, dst: torch.Tensor, first_eid: int, num_nodes: int, rank: int,
                    world: int, group=None):
    """Distributed build_compressed over torch.distributed (see above).
    Returns (cuts, CsrView of this rank's rows)."""
    deg = local_degrees(dst, num_nodes)
    if dist.get_backend(group) == "gloo":
        d = deg.cpu()
        dist.all_reduce(d, group=group)
        deg = d.to(deg.device)
    else:
        dist.all_reduce(deg, group=group)
    cuts = cuts_from_degrees(deg, world)
    s, d, e, counts = route_edges(src, dst, first_eid, cuts)
    rs, rd, re = _alltoall_rows([s, d, e], counts, group)
    del s, d, e
    return cuts, local_csc_from_routed(rs, rd, re, int(cuts[rank]), int(cuts[rank + 1]), num_nodes)


# ---------------------------------------------------------------------------
# Exchange-overlapped aggregation: the rank's rows are split
# by source into block 0 (sources in its own X shard: runs at once, while the
# exchange is in flight) and blocks 1..G (sources delivered by exchange chunk
# c: the all-gather of shard rows [c*CS, (c+1)*CS) from every rank). Each chunk
# is its own async all-gather; block c+1 runs as soon as chunk c has landed,
# continuing the rows' accumulation (gm_spmm_accumulate).
# ---------------------------------------------------------------------------
def chunk_layout(num_src_rows: int, world: int, chunks: int):
    """(shard_rows S, chunk_rows CS): shard q owns sources [q*S, (q+1)*S);
    exchange chunk c carries shard rows [c*CS, (c+1)*CS) of every rank."""
    s = -(-num_src_rows // world)
    return s, -(-s // chunks)


def source_blocks(num_src_rows: int, rank: int, world: int, chunks: int, device=None):
    """Per source id: (block, column inside that block's x).
    block 0: own shard, column = row inside x_shard;
    block 1+c: chunk c, column = q*CS + (o - c*CS) inside the chunk's gathered
    buffer [world*CS, F] (q = owner rank, o = row inside the owner's shard)."""
    s_rows, cs = chunk_layout(num_src_rows, world, chunks)
    s = torch.arange(num_src_rows, dtype=torch.int64, device=device)
    q = s // s_rows
    o = s - q * s_rows
    c = o // cs
    own = q == rank
    blk = torch.where(own, torch.zeros_like(c), 1 + c).to(torch.int32)
    col = torch.where(own, o, q * cs + (o - c * cs)).to(torch.int32)
    return blk, col


class _Done:
    def wait(self):
        return None


def _block_spmm(v, x, f, kind, out, arg, accumulate, mean_deg=None, carry=None, carry_mode=0, what="gm_spmm"):
    """One source block of a rank's rows: a fresh gm_spmm, a seeded
    gm_spmm_accumulate, or (bf16 sum/mean) gm_spmm_ex with the fp32 carry."""
    from .graphmill import _DT, _p, _stream
    lib = L.lib()
    cs = v.c_struct()
    plan = v.plan(f * x.element_size())
    dt = _DT[x.dtype]
    md = _p(mean_deg) if (mean_deg is not None and kind == L.GM_MEAN) else None
    if carry is not None:
        ep = L.gm_spmm_epilogue()
        ep.carry = carry.data_ptr()
        ep.carry_mode = carry_mode
        L.check(lib.gm_spmm_ex(C.byref(cs), C.byref(plan), dt, _p(x), f, None, kind, 1 if accumulate else 0, md,
                               C.byref(ep), _p(out), None, _stream()), what)
    elif accumulate:
        L.check(lib.gm_spmm_accumulate(C.byref(cs), C.byref(plan), dt, _p(x), f, None, kind, md, _p(out),
                                       _p(arg) if arg is not None else None, _stream()), what)
    else:
        L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), dt, _p(x), f, None, None, kind, _p(out),
                            _p(arg) if arg is not None else None, _stream()), what)


def _carry_buffer(cache, n, f, device):
    key = ("carry", n, f)
    if key not in cache:
        cache[key] = torch.empty(n, f, dtype=torch.float32, device=device)
    return cache[key]


class BlockedSpmm:
    """One rank's exchange-overlapped SpMM over its destination rows.

    rows: this rank's CSC row slice (CsrView, sources are global ids);
    x_shard passed to __call__: [chunks*CS, F] (this rank's X shard, zero
    padded). allgather(out, inp) -> work with .wait(): the chunk exchange
    (default: async NCCL all_gather_into_tensor). Results: MAX/MIN values and
    argmax equal the single-GPU ones bit-for-bit (NaN-free inputs); SUM/MEAN
    continue each row's sum across blocks (fp32-tolerance, one re-association
    per block boundary). bf16 SUM/MEAN carry the running rows in fp32
    (gm_spmm_ex GM_CARRY_*) and round once, in the last block, as one GPU does.
    For bit-identical sums use exact mode (allgather_features + one gm_spmm)."""

    def __init__(self, rows, num_src_rows: int, rank: int, world: int, chunks: int = 4,
                 allgather=None, group=None):
        from .graphmill import CsrView, _p, _stream
        self.rank, self.world, self.chunks = rank, world, chunks
        self.s_rows, self.cs = chunk_layout(num_src_rows, world, chunks)
        self.allgather = allgather or (lambda out, inp: dist.all_gather_into_tensor(
            out, inp, group=group, async_op=True))
        dev = rows.rowptr.device
        lib = L.lib()
        blk, colmap = source_blocks(num_src_rows, rank, world, chunks, dev)
        nb = chunks + 1
        n = rows.num_rows()
        nnz = rows.num_entries()
        self.rowptr_b = torch.empty(nb * (n + 1), dtype=torch.int64, device=dev)
        self.col_b = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        self.perm_b = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        wsb = lib.gm_csr_split_blocks_workspace(n, nb)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        cs = rows.c_struct()
        L.check(lib.gm_csr_split_blocks(C.byref(cs), _p(blk), _p(colmap), nb, _p(self.rowptr_b), _p(self.col_b),
                                        _p(self.perm_b), _p(ws), wsb, _stream()), "gm_csr_split_blocks")
        rp = self.rowptr_b.view(nb, n + 1)
        ends = rp[:, n].cpu().tolist()
        starts = rp[:, 0].cpu().tolist()
        self.blocks = []
        for b in range(nb):
            ncols = chunks * self.cs if b == 0 else world * self.cs
            self.blocks.append(CsrView(rp[b], self.col_b, self.perm_b, ncols, int(ends[b] - starts[b])))
        rr = rows.rowptr
        self.mean_deg = (rr[1:] - rr[:-1]).to(torch.int32)
        self._bufs = {}

    def block_nnz(self):
        return [v.num_entries() for v in self.blocks]

    def _buffers(self, f, dtype, device):
        key = (f, dtype)
        if key not in self._bufs:
            self._bufs[key] = [torch.empty(self.world * self.cs, f, dtype=dtype, device=device)
                               for _ in range(self.chunks)]
        return self._bufs[key]

    def __call__(self, x_shard: torch.Tensor, reduce: str = "sum", out: Optional[torch.Tensor] = None,
                 arg: Optional[torch.Tensor] = None):
        from .graphmill import _DT, _KIND, _p, _stream
        assert x_shard.shape[0] == self.chunks * self.cs, "x_shard must be padded to chunks*CS rows"
        x_shard = x_shard.contiguous()
        f = x_shard.shape[1]
        n = self.blocks[0].num_rows()
        maxmin = reduce in ("max", "min")
        carry = x_shard.dtype == torch.bfloat16 and not maxmin
        if out is None:
            out = torch.empty(n, f, dtype=x_shard.dtype, device=x_shard.device)
        if maxmin and arg is None:
            arg = torch.empty(n, f, dtype=torch.int32, device=x_shard.device)
        bufs = self._buffers(f, x_shard.dtype, x_shard.device)
        # every chunk's exchange is in flight before the local block starts
        works = [self.allgather(bufs[c], x_shard[c * self.cs:(c + 1) * self.cs]) or _Done()
                 for c in range(self.chunks)]
        first_kind = L.GM_SUM if reduce == "mean" else _KIND[reduce]
        # bf16 sums: fp32 running rows, rounded once in the last block (as one GPU)
        acc = _carry_buffer(self._bufs, n, f, x_shard.device) if carry else None
        _block_spmm(self.blocks[0], x_shard, f, first_kind, out, arg if maxmin else None, False,
                    carry=acc, carry_mode=L.GM_CARRY_START, what="gm_spmm (local block)")
        for c in range(self.chunks):
            works[c].wait()
            last = c == self.chunks - 1
            kind = _KIND[reduce] if (last or reduce != "mean") else L.GM_SUM
            _block_spmm(self.blocks[1 + c], bufs[c], f, kind, out, arg if maxmin else None, True,
                        mean_deg=self.mean_deg, carry=acc,
                        carry_mode=L.GM_CARRY_FINISH if last else L.GM_CARRY_CONTINUE, what="gm_spmm (block)")
        return (out, arg) if maxmin else out


# ---------------------------------------------------------------------------
# Halo-only exchange (SURVEY.md §8e "halo-only variant"): a rank receives only
# the source rows its destination rows actually reference, per peer, with one
# all_to_all_single per step instead of all-gathering every shard. The
# own-shard block aggregates while the exchange is in flight; the halo block
# (sources remapped into the receive buffer) continues the rows afterwards.
# ---------------------------------------------------------------------------
def halo_need(rows, num_src_rows: int, rank: int, world: int):
    """Per peer q: the ascending rows (indices inside q's X shard) that this
    rank's destination rows reference (own shard: empty). Device int32."""
    from .graphmill import _p, _stream
    s_rows = -(-num_src_rows // world)
    mark = torch.empty(num_src_rows, dtype=torch.uint8, device=rows.rowptr.device)
    cs = rows.c_struct()
    L.check(L.lib().gm_mark_columns(C.byref(cs), _p(mark), _stream()), "gm_mark_columns")
    ids = torch.nonzero(mark, as_tuple=True)[0]
    need = []
    for q in range(world):
        if q == rank:
            need.append(torch.empty(0, dtype=torch.int32, device=mark.device))
            continue
        sel = ids[(ids >= q * s_rows) & (ids < (q + 1) * s_rows)]
        need.append((sel - q * s_rows).to(torch.int32))
    return need


def exchange_need_lists(need, group=None):
    """all_to_all of the need lists: returns send[q] = the rows of MY shard
    that rank q needs (what I pack for q every step)."""
    world = len(need)
    dev = need[0].device
    counts = torch.tensor([t.numel() for t in need], dtype=torch.int64, device=dev)
    peer_counts = torch.empty_like(counts)
    dist.all_to_all_single(peer_counts, counts, group=group)
    pc = peer_counts.cpu().tolist()
    out = torch.empty(sum(pc), dtype=torch.int32, device=dev)
    dist.all_to_all_single(out, torch.cat(need) if need else out, output_split_sizes=pc,
                           input_split_sizes=[t.numel() for t in need], group=group)
    return list(torch.split(out, pc))


def halo_blocks(need, num_src_rows: int, rank: int, world: int, device=None):
    """(block, column) per source id for the halo layout: own shard -> block 0
    at its shard row; a needed row of peer q -> block 1 at its position in the
    receive buffer (peers in rank order, each peer's rows ascending)."""
    s_rows = -(-num_src_rows // world)
    blk = torch.full((num_src_rows,), 1, dtype=torch.int32, device=device)
    col = torch.zeros(num_src_rows, dtype=torch.int32, device=device)
    lo, hi = rank * s_rows, min((rank + 1) * s_rows, num_src_rows)
    blk[lo:hi] = 0
    col[lo:hi] = torch.arange(hi - lo, dtype=torch.int32, device=device)
    off = 0
    for q in range(world):
        n = need[q].numel()
        if q != rank and n:
            col[q * s_rows + need[q].long()] = torch.arange(off, off + n, dtype=torch.int32, device=device)
        off += n
    return blk, col


class HaloSpmm:
    """One rank's halo-exchange SpMM: block 0 (own shard) runs while the
    all_to_all of the packed halo rows is in flight; block 1 (the halo rows)
    continues every row with gm_spmm_accumulate. Numerics as BlockedSpmm
    (max/min + argmax exact, sum continued across one block boundary).

    need: halo_need(...) of this rank; send: exchange_need_lists(need) (rows of
    my shard each peer needs). alltoall(recv, send, recv_splits, send_splits)
    -> work (default: async NCCL all_to_all_single)."""

    def __init__(self, rows, num_src_rows: int, rank: int, world: int, need, send, alltoall=None, group=None):
        from .graphmill import CsrView, _p, _stream
        self.rank, self.world = rank, world
        self.s_rows = -(-num_src_rows // world)
        self.recv_splits = [int(t.numel()) for t in need]
        self.send_splits = [int(t.numel()) for t in send]
        self.send_idx = torch.cat(send) if send else torch.empty(0, dtype=torch.int32)
        self.alltoall = alltoall or (lambda r, s, rs, ss: dist.all_to_all_single(
            r, s, output_split_sizes=rs, input_split_sizes=ss, group=group, async_op=True))
        dev = rows.rowptr.device
        blk, colmap = halo_blocks(need, num_src_rows, rank, world, dev)
        n, nnz = rows.num_rows(), rows.num_entries()
        lib = L.lib()
        self.rowptr_b = torch.empty(2 * (n + 1), dtype=torch.int64, device=dev)
        self.col_b = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        self.perm_b = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        wsb = lib.gm_csr_split_blocks_workspace(n, 2)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        cs = rows.c_struct()
        L.check(lib.gm_csr_split_blocks(C.byref(cs), _p(blk), _p(colmap), 2, _p(self.rowptr_b), _p(self.col_b),
                                        _p(self.perm_b), _p(ws), wsb, _stream()), "gm_csr_split_blocks")
        rp = self.rowptr_b.view(2, n + 1)
        ends, starts = rp[:, n].cpu().tolist(), rp[:, 0].cpu().tolist()
        halo_rows = sum(self.recv_splits)
        self.blocks = [CsrView(rp[0], self.col_b, self.perm_b, self.s_rows, int(ends[0] - starts[0])),
                       CsrView(rp[1], self.col_b, self.perm_b, max(halo_rows, 1), int(ends[1] - starts[1]))]
        rr = rows.rowptr
        self.mean_deg = (rr[1:] - rr[:-1]).to(torch.int32)
        self._bufs = {}

    def halo_rows(self) -> int:
        return sum(self.recv_splits)

    def __call__(self, x_shard: torch.Tensor, reduce: str = "sum", out: Optional[torch.Tensor] = None,
                 arg: Optional[torch.Tensor] = None):
        from .graphmill import _DT, _KIND, _p, _stream
        x_shard = x_shard.contiguous()
        f = x_shard.shape[1]
        n = self.blocks[0].num_rows()
        maxmin = reduce in ("max", "min")
        carry = x_shard.dtype == torch.bfloat16 and not maxmin
        if out is None:
            out = torch.empty(n, f, dtype=x_shard.dtype, device=x_shard.device)
        if maxmin and arg is None:
            arg = torch.empty(n, f, dtype=torch.int32, device=x_shard.device)
        key = (f, x_shard.dtype)
        if key not in self._bufs:
            self._bufs[key] = (torch.empty(max(self.send_idx.numel(), 1), f, dtype=x_shard.dtype, device=x_shard.device),
                               torch.empty(max(self.halo_rows(), 1), f, dtype=x_shard.dtype, device=x_shard.device))
        send_buf, recv_buf = self._bufs[key]
        lib = L.lib()
        dt = _DT[x_shard.dtype]
        # pack what every peer needs from my shard, then exchange
        L.check(lib.gm_gather_rows(dt, _p(x_shard), f, _p(self.send_idx), self.send_idx.numel(), _p(send_buf),
                                   _stream()), "gm_gather_rows")
        work = self.alltoall(recv_buf[: self.halo_rows()], send_buf[: self.send_idx.numel()], self.recv_splits,
                             self.send_splits) or _Done()
        first_kind = L.GM_SUM if reduce == "mean" else _KIND[reduce]
        acc = _carry_buffer(self._bufs, n, f, x_shard.device) if carry else None
        _block_spmm(self.blocks[0], x_shard, f, first_kind, out, arg if maxmin else None, False,
                    carry=acc, carry_mode=L.GM_CARRY_START, what="gm_spmm (own shard)")
        work.wait()
        _block_spmm(self.blocks[1], recv_buf, f, _KIND[reduce], out, arg if maxmin else None, True,
                    mean_deg=self.mean_deg, carry=acc, carry_mode=L.GM_CARRY_FINISH, what="gm_spmm (halo)")
        return (out, arg) if maxmin else out


# ---------------------------------------------------------------------------
# Push mode: the exchange of layer l+1 fused into the SpMM of layer l. Every
# rank keeps a replica of the layer input X ([N, F]); the SpMM over its
# destination rows reads the local replica only and its epilogue stores each
# finished output row both into its own next-layer replica and, over NVLink
# P2P, into every peer's replica that references the row (gm_spmm_ex push).
# No collective moves features: a one-element all_reduce after the kernel
# orders the peers' next reads. Rows are computed by the single-GPU kernel
# over the whole local X, so results are bit-identical to one GPU.
# ---------------------------------------------------------------------------
def push_masks(rows, num_src_rows: int, r0: int, r1: int, rank: int, world: int, gather=None, group=None):
    """Per local row v in [r0, r1): bit j set iff the j-th peer (ranks in
    order, this rank skipped) references source v. gather(t) -> [world, N] stack of every rank's referenced-column
    bitmap (default: all_gather over `group`). uint32 [r1 - r0] on the device."""
    from .graphmill import _p, _stream
    mark = torch.empty(num_src_rows, dtype=torch.uint8, device=rows.rowptr.device)
    cs = rows.c_struct()
    L.check(L.lib().gm_mark_columns(C.byref(cs), _p(mark), _stream()), "gm_mark_columns")
    if gather is None:
        parts = [torch.empty_like(mark) for _ in range(world)]
        dist.all_gather(parts, mark, group=group)
        allm = torch.stack(parts)
    else:
        allm = gather(mark)
    return masks_from_bitmaps(allm, r0, r1, rank)


def masks_from_bitmaps(allm: torch.Tensor, r0: int, r1: int, rank: int) -> torch.Tensor:
    """allm [world, N]: every rank's referenced-source bitmap. Per row of
    [r0, r1): bit j = the j-th peer in rank order without `rank` (PushSpmm's
    push_dst[j]) references it."""
    world = allm.shape[0]
    bits = (allm[:, r0:r1].to(torch.int64) != 0).to(torch.int64)
    w = torch.tensor([0 if q == rank else 1 << (q if q < rank else q - 1) for q in range(world)],
                     dtype=torch.int64, device=bits.device).view(world, 1)
    return (bits * w).sum(0).to(torch.int32).contiguous()


def open_peer_buffers(t: torch.Tensor, group=None):
    """Map every peer's `t` (same shape on every rank) into this process over
    CUDA IPC (NVLink P2P). Returns [world] device pointers (own rank: t's
    pointer) and the opened bases to close with close_peer_buffers."""
    lib = L.lib()
    nb = lib.gm_ipc_handle_bytes()
    h = (C.c_ubyte * nb)()
    L.check(lib.gm_ipc_get_handle(C.c_void_p(t.data_ptr()), h), "gm_ipc_get_handle")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h), group=group)
    ptrs, bases = [], []
    for q in range(world):
        if q == rank:
            ptrs.append(t.data_ptr())
            continue
        buf = (C.c_ubyte * nb).from_buffer_copy(handles[q])
        p, b = C.c_void_p(), C.c_void_p()
        L.check(lib.gm_ipc_open_handle(buf, C.byref(p), C.byref(b)), "gm_ipc_open_handle")
        ptrs.append(p.value)
        bases.append(b.value)
    return ptrs, bases


def close_peer_buffers(bases):
    for b in bases:
        L.check(L.lib().gm_ipc_close_handle(C.c_void_p(b)), "gm_ipc_close_handle")


class PushSpmm:
    """One rank's push-mode SpMM over its destination rows [r0, r1).

    rows: the rank's CSC row slice (global source ids); mask: push_masks(...)
    or None (push every row to every peer). __call__(x, out_next, peer_ptrs)
    reads x (this rank's full replica of the layer input), writes the rows to
    out_next[r0:r1] and pushes them into peer_ptrs[q] ([N, F] replicas of the
    next layer's input on the other ranks, peer_ptrs[rank] ignored)."""

    def __init__(self, rows, r0: int, r1: int, rank: int, world: int, mask: Optional[torch.Tensor] = None):
        assert world - 1 <= L.GM_MAX_PUSH, "push mode targets at most GM_MAX_PUSH peers"
        self.rows, self.r0, self.r1, self.rank, self.world, self.mask = rows, r0, r1, rank, world, mask

    def __call__(self, x: torch.Tensor, out_next: torch.Tensor, peer_ptrs, reduce: str = "sum",
                 arg: Optional[torch.Tensor] = None):
        """max/min: the values are pushed; the argmax of this rank's rows goes
        to `arg` ([r1 - r0, F] int32, allocated when None) and is returned."""
        from .graphmill import _DT, _KIND, _p, _stream
        maxmin = reduce in ("max", "min")
        f = x.shape[1]
        if maxmin and arg is None:
            arg = torch.empty(self.r1 - self.r0, f, dtype=torch.int32, device=x.device)
        lib = L.lib()
        ep = L.gm_spmm_epilogue()
        n = 0
        for q in range(self.world):
            if q != self.rank:
                ep.push_dst[n] = peer_ptrs[q]
                n += 1
        ep.n_push = n
        ep.push_row0 = self.r0
        ep.push_mask = self.mask.data_ptr() if self.mask is not None else None
        cs = self.rows.c_struct()
        plan = self.rows.plan(f * x.element_size())
        L.check(lib.gm_spmm_ex(C.byref(cs), C.byref(plan), _DT[x.dtype], _p(x), f, None, _KIND[reduce], 0, None,
                               C.byref(ep), _p(out_next[self.r0:self.r1]), _p(arg) if maxmin else None, _stream()),
                "gm_spmm_ex (push)")
        return (out_next, arg) if maxmin else out_next


# ---------------------------------------------------------------------------
# The same three modes through the library's own C-ABI over NCCL
# (gm_dist_spmm): the exchange is issued by the library on a comm stream and
# each source block waits on a device event for just its chunk — no host
# synchronisation per step. The communicator is NCCL's own (bootstrapped here
# over torch.distributed); a C++ host passes its ncclComm_t directly.
# ---------------------------------------------------------------------------
class NcclComm:
    """An NCCL communicator created through gm_nccl_comm_init; the 128-byte
    unique id travels over the torch.distributed group (any backend)."""

    def __init__(self, rank: int, world: int, group=None):
        lib = L.lib()
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            L.check(lib.gm_nccl_unique_id(C.cast(uid, C.c_void_p)), "gm_nccl_unique_id")
        if world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            C.memmove(uid, box[0], 128)
        self.comm = C.c_void_p()
        L.check(lib.gm_nccl_comm_init(world, C.cast(uid, C.c_void_p), rank, C.byref(self.comm)), "gm_nccl_comm_init")
        self.rank, self.world = rank, world

    def close(self):
        if self.comm:
            L.check(L.lib().gm_nccl_comm_destroy(self.comm), "gm_nccl_comm_destroy")
            self.comm = C.c_void_p()


class DistSpmm:
    """One rank's partitioned SpMM through gm_dist_spmm.

    mode "exact": view = the rank's row slice with global source ids;
    "blocked": view split into 1 + chunks source blocks (as BlockedSpmm);
    "halo": need = halo_need(...), send = exchange_need_lists(need)."""

    def __init__(self, rows, num_src_rows: int, comm: NcclComm, mode: str = "blocked", chunks: int = 4,
                 need=None, send=None):
        from .graphmill import CsrView, _p, _stream
        self.comm, self.mode = comm, mode
        rank, world = comm.rank, comm.world
        self.rank, self.world = rank, world
        lib = L.lib()
        dev = rows.rowptr.device
        n, nnz = rows.num_rows(), rows.num_entries()
        self.s_rows = -(-num_src_rows // world)
        self._keep = []
        if mode == "exact":
            views = [rows]
            self.chunks, self.cs = 0, 0
        else:
            if mode == "blocked":
                self.chunks = chunks
                self.s_rows, self.cs = chunk_layout(num_src_rows, world, chunks)
                blk, colmap = source_blocks(num_src_rows, rank, world, chunks, dev)
                nb = chunks + 1
            elif mode == "halo":
                self.chunks, self.cs = 0, 0
                blk, colmap = halo_blocks(need, num_src_rows, rank, world, dev)
                nb = 2
            else:
                raise ValueError(f"DistSpmm: unknown mode {mode}")
            rowptr_b = torch.empty(nb * (n + 1), dtype=torch.int64, device=dev)
            col_b = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
            perm_b = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
            wsb = lib.gm_csr_split_blocks_workspace(n, nb)
            ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
            cs = rows.c_struct()
            L.check(lib.gm_csr_split_blocks(C.byref(cs), _p(blk), _p(colmap), nb, _p(rowptr_b), _p(col_b),
                                            _p(perm_b), _p(ws), wsb, _stream()), "gm_csr_split_blocks")
            rp = rowptr_b.view(nb, n + 1)
            ends, starts = rp[:, n].cpu().tolist(), rp[:, 0].cpu().tolist()
            views = []
            for b in range(nb):
                if mode == "blocked":
                    ncols = chunks * self.cs if b == 0 else world * self.cs
                else:
                    ncols = self.s_rows if b == 0 else max(1, sum(int(t.numel()) for t in need))
                views.append(CsrView(rp[b], col_b, perm_b, ncols, int(ends[b] - starts[b])))
            self._keep += [rowptr_b, col_b, perm_b]
        self.views = views
        self.mean_deg = (rows.rowptr[1:] - rows.rowptr[:-1]).to(torch.int32)
        self._ws = {}
        self.comm_stream = torch.cuda.Stream(device=dev)
        lay = L.gm_dist_layout()
        lay.rank, lay.world = rank, world
        lay.mode = {"exact": L.GM_DIST_EXACT, "blocked": L.GM_DIST_BLOCKED, "halo": L.GM_DIST_HALO}[mode]
        lay.chunks = self.chunks
        lay.shard_rows = self.s_rows
        lay.chunk_rows = self.cs
        self._blocks = (L.gm_csr * len(views))(*[v.c_struct() for v in views])
        lay.blocks = self._blocks
        lay.mean_deg = self.mean_deg.data_ptr()
        if mode == "halo":
            self.send_idx = torch.cat(send).to(torch.int32) if send else torch.empty(0, dtype=torch.int32, device=dev)
            self._send_counts = (C.c_int64 * world)(*[int(t.numel()) for t in send])
            self._recv_counts = (C.c_int64 * world)(*[int(t.numel()) for t in need])
            lay.halo_send_idx = self.send_idx.data_ptr() if self.send_idx.numel() else None
            lay.halo_send_counts_host = self._send_counts
            lay.halo_recv_counts_host = self._recv_counts
        self.layout = lay
        self._plans = {}

    def _plans_for(self, row_bytes):
        key = 4096 if row_bytes >= 1024 else 0
        if key not in self._plans:
            self._plans[key] = (L.gm_spmm_plan * len(self.views))(*[v.plan(row_bytes) for v in self.views])
        return self._plans[key]

    def __call__(self, x_shard: torch.Tensor, reduce: str = "sum", out: Optional[torch.Tensor] = None,
                 arg: Optional[torch.Tensor] = None):
        from .graphmill import _DT, _KIND, _p, _stream
        x_shard = x_shard.contiguous()
        f = x_shard.shape[1]
        n = self.views[0].num_rows()
        maxmin = reduce in ("max", "min")
        if out is None:
            out = torch.empty(n, f, dtype=x_shard.dtype, device=x_shard.device)
        if maxmin and arg is None:
            arg = torch.empty(n, f, dtype=torch.int32, device=x_shard.device)
        self.layout.plans = self._plans_for(f * x_shard.element_size())
        key = (f, x_shard.dtype)
        lib = L.lib()
        if key not in self._ws:
            nb = lib.gm_dist_spmm_workspace(C.byref(self.layout), _DT[x_shard.dtype], f)
            self._ws[key] = torch.empty(max(nb, 1), dtype=torch.uint8, device=x_shard.device)
        ws = self._ws[key]
        L.check(lib.gm_dist_spmm(C.byref(self.layout), _DT[x_shard.dtype], _p(x_shard), f, _KIND[reduce], _p(out),
                                 _p(arg) if maxmin else None, _p(ws), ws.numel(), self.comm.comm,
                                 C.c_void_p(self.comm_stream.cuda_stream), _stream()), "gm_dist_spmm")
        return (out, arg) if maxmin else out
