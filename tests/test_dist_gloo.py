"""N>1 host logic on CPU: world_size-2 gloo processes run the real partitioner
(gm_partition_rows_by_nnz from the C-ABI library) and the real exchange
(all_gather_into_tensor), then aggregate their destination-row slice with the
oracle restatement (the only CPU stand-in for the device kernel, which cannot
run here). The concatenated per-rank outputs must equal the single-process
oracle bit-for-bit — the property that makes the GPU path correct by
construction (per-row results never depend on the partition)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, e, f, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2507_16991_b200 import _lib as L
        from paper_2507_16991_b200.dist import allgather_features, make_shard
        lib = L.lib()
        src = np.zeros(e, np.int64)
        dst = np.zeros(e, np.int64)
        lib.gm_synth_edges_host(1, 99, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
        orc = Oracle()
        rp, col, perm = orc.build_compressed(dst, src, n)
        sh = make_shard(rp, n, rank, world)
        # this rank's X shard (rows it owns), produced locally
        x = np.zeros((n, f), np.float32)
        lib.gm_synth_features_host(99, 0, n, f, 1, L.GM_F32, x.ctypes.data)
        lo, hi = sh.x_rows()
        shard = np.zeros((sh.shard_rows, f), np.float32)
        shard[: max(0, min(hi, n) - lo)] = x[lo:min(hi, n)]
        full = allgather_features(torch.from_numpy(shard), sh).numpy()[:n]
        assert full.tobytes() == x.tobytes()
        rows = np.arange(sh.row_begin, sh.row_end)
        out = orc.spmm(rp, col, perm, full, rows=rows)
        mx, arg = orc.spmm_max(rp, col, perm, full, rows=rows)
        q.put((rank, sh.row_begin, sh.row_end, out, mx, arg, int(rp[sh.row_end] - rp[sh.row_begin])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_spmm_matches_single_process(world):
    n, e, f = 3000, 60000, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, e, f, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    from paper_2507_16991_b200 import _lib as L
    lib = L.lib()
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    lib.gm_synth_edges_host(1, 99, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    x = np.zeros((n, f), np.float32)
    lib.gm_synth_features_host(99, 0, n, f, 1, L.GM_F32, x.ctypes.data)
    orc = Oracle()
    rp, col, perm = orc.build_compressed(dst, src, n)
    want = orc.spmm(rp, col, perm, x)
    wmx, warg = orc.spmm_max(rp, col, perm, x)
    # contiguous, covering, nnz-balanced
    assert results[0][1] == 0 and results[-1][2] == n
    for a, b in zip(results, results[1:]):
        assert a[2] == b[1]
    loads = [r[6] for r in results]
    assert max(loads) - min(loads) <= max(rp[1:] - rp[:-1]) + 1
    got = np.concatenate([r[3] for r in results])
    assert got.tobytes() == want.tobytes()
    assert np.concatenate([r[4] for r in results]).tobytes() == wmx.tobytes()
    assert np.array_equal(np.concatenate([r[5] for r in results]), warg)


def _chunk_worker(rank, world, port, n, f, chunks, q):
    """Chunked exchange of BlockedSpmm: every source id's (block, column)
    must address exactly its feature row — in the own shard (block 0) or in
    the gathered chunk buffer (block 1+c)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_16991_b200.dist import chunk_layout, source_blocks
        s_rows, cs = chunk_layout(n, world, chunks)
        x = torch.arange(n * f, dtype=torch.float32).view(n, f)
        shard = torch.zeros(chunks * cs, f)
        lo, hi = rank * s_rows, min((rank + 1) * s_rows, n)
        shard[: max(0, hi - lo)] = x[lo:hi]
        bufs = [torch.empty(world * cs, f) for _ in range(chunks)]
        works = [dist.all_gather_into_tensor(bufs[c], shard[c * cs:(c + 1) * cs], async_op=True)
                 for c in range(chunks)]
        for w in works:
            w.wait()
        blk, col = source_blocks(n, rank, world, chunks)
        ok = True
        for s in range(n):
            b, c = int(blk[s]), int(col[s])
            row = shard[c] if b == 0 else bufs[b - 1][c]
            ok &= bool(torch.equal(row, x[s]))
            ok &= (b == 0) == (lo <= s < hi)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks", [(2, 3), (3, 2)])
def test_chunked_exchange_addresses_every_source(world, chunks):
    n, f = 1001, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, world, port, n, f, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


def _halo_worker(rank, world, port, n, f, q):
    """Halo protocol on gloo: need lists exchanged with all_to_all, rows packed
    per peer (index_select stands in for gm_gather_rows on CPU) and exchanged
    with all_to_all_single; every referenced remote source must land at the
    column halo_blocks assigns it."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_16991_b200.dist import exchange_need_lists, halo_blocks
        rng = np.random.default_rng(100 + rank)
        s_rows = -(-n // world)
        refd = np.unique(rng.integers(0, n, 700))
        need = []
        for p in range(world):
            sel = refd[(refd >= p * s_rows) & (refd < min((p + 1) * s_rows, n))] - p * s_rows
            need.append(torch.from_numpy(sel.astype(np.int32)) if p != rank else torch.empty(0, dtype=torch.int32))
        send = exchange_need_lists(need)
        x = torch.arange(n * f, dtype=torch.float32).view(n, f)
        lo, hi = rank * s_rows, min((rank + 1) * s_rows, n)
        shard = x[lo:hi]
        packed = torch.cat([shard[s.long()] for s in send]) if sum(s.numel() for s in send) else torch.empty(0, f)
        recv = torch.empty(sum(t.numel() for t in need), f)
        dist.all_to_all_single(recv, packed, output_split_sizes=[t.numel() for t in need],
                               input_split_sizes=[s.numel() for s in send])
        blk, col = halo_blocks(need, n, rank, world)
        ok = True
        for s in refd.tolist():
            b, c = int(blk[s]), int(col[s])
            row = shard[c] if b == 0 else recv[c]
            ok &= bool(torch.equal(row, x[s]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_protocol_addresses_every_referenced_source(world):
    n, f = 3001, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, n, f, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


def _build_worker(rank, world, port, n, e, q):
    """Distributed build_compressed protocol on gloo (dist.build_local_csc's
    collectives and ordering argument): degree all-reduce, the real nnz
    partitioner, owner routing through dist._alltoall_rows (gloo path), then
    the local stable build — the oracle's counting sort stands in for the
    device kernels (stable grouping by owner, local compress)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2507_16991_b200 import _lib as L
        from paper_2507_16991_b200.dist import _alltoall_rows, partition_rows_by_nnz
        lib = L.lib()
        e0, e1 = rank * e // world, (rank + 1) * e // world
        src = np.zeros(e1 - e0, np.int64)
        dst = np.zeros(e1 - e0, np.int64)
        lib.gm_synth_edges_host(1, 5, e0, e1 - e0, n, n, src.ctypes.data, dst.ctypes.data)
        deg = torch.from_numpy(np.bincount(dst, minlength=n).astype(np.int32))
        dist.all_reduce(deg)
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(deg.numpy().astype(np.int64), out=rp[1:])
        cuts = partition_rows_by_nnz(rp, world)
        owner = np.searchsorted(cuts[1:], dst, side="right")
        order = np.argsort(owner, kind="stable")
        counts = np.bincount(owner, minlength=world).tolist()
        rs, rd, re = _alltoall_rows([torch.from_numpy(src[order]), torch.from_numpy(dst[order]),
                                     torch.from_numpy(order + e0)], counts)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        lrp, lcol, lperm = Oracle().build_compressed(rd.numpy() - r0, rs.numpy(), r1 - r0)
        q.put((rank, r0, r1, lrp, lcol, re.numpy()[lperm]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_build_protocol_matches_global_csc(world):
    n, e = 3000, 60000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_build_worker, args=(r, world, port, n, e, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    from paper_2507_16991_b200 import _lib as L
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    L.lib().gm_synth_edges_host(1, 5, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    rp, col, perm = Oracle().build_compressed(dst, src, n)
    covered = 0
    for rank, r0, r1, lrp, lcol, lperm in sorted(res, key=lambda t: t[0]):
        assert np.array_equal(lrp, rp[r0:r1 + 1] - rp[r0])
        assert np.array_equal(lcol, col[rp[r0]:rp[r1]])
        assert np.array_equal(lperm, perm[rp[r0]:rp[r1]])
        covered += r1 - r0
    assert covered == n


def test_push_mask_bits_name_the_peer_slots():
    from paper_2507_16991_b200.dist import masks_from_bitmaps
    allm = torch.tensor([[1, 0, 1, 1], [0, 1, 1, 0], [1, 1, 0, 1]], dtype=torch.uint8)  # 3 ranks, 4 rows
    # rank 1 owns rows [1, 3); its peers in push_dst order are ranks 0, 2 -> bits 0, 1
    m = masks_from_bitmaps(allm, 1, 3, 1)
    assert m.tolist() == [0b10, 0b01]
    # rank 0 owns rows [0, 2); peers 1, 2 -> bits 0, 1
    assert masks_from_bitmaps(allm, 0, 2, 0).tolist() == [0b10, 0b11]
