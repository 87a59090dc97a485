#!/usr/bin/env python3
"""bench.py — headline benchmark of the CSR SpMM aggregation hot path on B200.

Workload (BASELINE.json configs[3], the configuration the metric is quoted on):
ogbn-products-shaped power-law graph, N = 2,449,029 nodes, E = 61,859,140
edges (Chung-Lu alpha = 0.5, ids permuted), F = 100 fp32 features, full-graph
sum aggregation (the reference's spmm(e, x, nullopt, sum), message_passing.hpp:92).
A "step" is one full-graph SpMM over the resident graph (the CSC and its plan
are cached like the reference's EdgeIndex cache and built outside the timed
region). Synthetic data (no network); X (980 MB) is larger than L2 (126 MB).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): destination rows are nnz-partitioned across ranks, X is
row-sharded and all-gathered over NCCL every step (the exchange a multi-layer
model needs), then each rank aggregates its rows; time = max over ranks.
`--impl reference` times the reference's own CPU spmm (oracle/_ref, compiled
in place from /root/reference) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GEdges/s CSR SpMM aggr (frac of HBM BW) + segment_matmul TFLOP/s @1/2/4/8 B200"
N_NODES, N_EDGES, F = 2_449_029, 61_859_140, 100
SEED = 0x67726170686D696C  # derive(..) base seed of SURVEY §8d ("graphmil")
CHUNKS = 4  # exchange chunks per step at N > 1 (BlockedSpmm)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def spmm_bytes(n_dst, e, f, esz=4):
    """Gather-model algorithmic bytes of one sum SpMM:
    E*(F*s + 4 col) + N*(8 rowptr + F*s out)."""
    return e * (f * esz + 4) + n_dst * (8 + f * esz)


def make_graph(gm, L, n, e, f, device, stream):
    src = torch.empty(e, dtype=torch.int64, device=device)
    dst = torch.empty(e, dtype=torch.int64, device=device)
    L.check(L.lib().gm_synth_edges(1, SEED, 0, e, n, n, src.data_ptr(), dst.data_ptr(), stream))
    x = torch.empty(n, f, dtype=torch.float32, device=device)
    L.check(L.lib().gm_synth_features(SEED, 0, n, f, 0, L.GM_F32, x.data_ptr(), stream))
    g = gm.EdgeIndex(src, dst, n, n, device=device)
    return g, x


def bench_segment_matmul(gm, L, device, f=128, rows=1_939_743, rank=0, world=1, dist=None, fp32=False):
    """Node-type segment_matmul, K = N = f, bf16 in/out. f=128: C3 (OGB-MAG)
    with the real per-type row counts; larger f: the tensor-bound F-sweep.
    fp32=True: the reference's dtype, fp32 in/out through the fused 3-piece
    split (six bf16 products per MAC: tensor ceiling = bf16 peak / 6).
    world > 1: W replicated, every group's rows split evenly
    across ranks, no collective; time = max over ranks, TFLOP/s of the whole job."""
    if f == 128 and rows == 1_939_743:
        gptr = [0, 736_389, 1_871_038, 1_879_778, 1_939_743]
    else:
        gptr = [0, rows * 38 // 100, rows * 96 // 100, rows * 97 // 100, rows]
    total_rows = gptr[-1]
    ptr = [0]
    for g in range(4):
        m = gptr[g + 1] - gptr[g]
        ptr.append(ptr[-1] + (m * (rank + 1)) // world - (m * rank) // world)
    x = torch.randn(ptr[-1], f, device=device).to(torch.bfloat16)
    w = (torch.randn(4, f, f, device=device) / f ** 0.5).to(torch.bfloat16)
    if fp32:
        x, w = x.float(), w.float()
    esz, tscale = (4, 6) if fp32 else (2, 1)
    try:
        for _ in range(3):
            gm.segment_matmul(x, ptr, w)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 20
        ev[0].record()
        for _ in range(reps):
            gm.segment_matmul(x, ptr, w)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
    except Exception as exc:  # reported, never silently substituted
        return {"error": str(exc)[:200]}
    if dist is not None:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = 2.0 * total_rows * f * f
    byts = 2.0 * total_rows * f * esz + world * 4 * f * f * esz
    hbm, bf16_peak, _ = peaks()
    ai = flops / byts
    hbm, bf16_peak = hbm * world, bf16_peak * world / tscale
    ceiling = min(bf16_peak, ai * hbm / 1e3)
    return {"shape": f"sum_M={total_rows},K=N={f},G=4,{'fp32' if fp32 else 'bf16'}", "n_gpus": world, "ms": ms, "tflops": flops / ms / 1e9,
            "frac_tensor_peak": flops / ms / 1e9 / bf16_peak, "achieved_gbs": byts / ms / 1e6,
            "frac_hbm": byts / ms / 1e6 / hbm, "roofline_ceiling_tflops": ceiling,
            "frac_roofline": flops / ms / 1e9 / ceiling,
            "bound": "hbm" if ai * hbm / 1e3 < bf16_peak else "tensor"}


def workload_config(world: int) -> dict:
    """The `config` both arms print (same workload, same keys)."""
    return {"workload": "ogbn-products-shaped power-law graph (configs[3]), full-graph sum SpMM",
            "nodes": N_NODES, "edges": N_EDGES, "feats": F, "graph": "Chung-Lu alpha=0.5",
            "seed": hex(SEED),
            "parallelism": f"dst-row partition x{world}" + (
                f" + {CHUNKS} chunked async NCCL all-gathers of X overlapped with source-blocked "
                "aggregation" if world > 1 else ""),
            "l2": "GPU arm: L2 flushed between timed steps (256 MB write); X = 980 MB > L2"}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU spmm<float> (oracle/_ref, the
    unmodified reference compiled in place) on this host, rank 0 only. Inputs
    come from the oracle-side generator (ref_synth_*, the reference's rng::Stream),
    so this arm never loads the product library. Each step is one full-graph
    sum SpMM over all host threads (row ranges, one reference spmm per thread);
    single-core lines (the reference's own single-threaded convention,
    message_passing.hpp:676-697) are reported beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import Reference, cpu_model, host_threads
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    ref = Reference()
    threads = host_threads()
    src, dst = ref.synth_edges(1, SEED, N_EDGES, N_NODES, N_NODES, threads=threads)
    x = ref.synth_features(SEED, N_NODES, F, threads=threads)
    secs, edges = ref.bench_spmm(src, dst, N_NODES, N_NODES, x, mean=False, threads=threads,
                                 rows_limit=0, warmup=args.warmup, repeat=args.steps)
    assert edges == N_EDGES
    val = edges / secs / 1e9
    # single-core lines ("1 of N cores"): spmm and the max path on a 1/16 row
    # sample, build_compressed of the full CSC
    rows = N_NODES // 16
    s1, e1 = ref.bench_spmm(src, dst, N_NODES, N_NODES, x, threads=1, rows_limit=rows, warmup=1, repeat=2)
    m1, em = ref.bench_max(src, dst, N_NODES, N_NODES, x, rows_limit=rows)
    b1 = ref.bench_build_compressed(dst, src, N_NODES)
    model = cpu_model()
    sample = (f"full graph ({edges} edges) per step: reference spmm<float> sum, {threads} threads "
              f"over dst-row ranges (one reference spmm per thread), CSC caches filled outside the timed region")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GEdges/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.gpus),
        "cpu_baseline": {"value": val, "unit": "GEdges/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": model},
        "e2e": {"value": val, "unit": "GEdges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "single_core": {
            "cpu_model": model, "cores": f"1 of {threads}",
            "spmm_sum": {"gedges_s": e1 / s1 / 1e9, "ms": s1 * 1e3,
                         "sample": f"dst rows [0,{rows}) ({e1} edges)"},
            "max_path": {"gedges_s": em / m1 / 1e9, "ms": m1 * 1e3,
                         "sample": f"dst rows [0,{rows}) ({em} edges), dst_grouped_order + gather_rows + "
                                   "aggregate(max)"},
            "build_compressed_csc": {"gedges_s": N_EDGES / b1 / 1e9, "ms": b1 * 1e3,
                                     "sample": f"full graph ({N_EDGES} edges)"}},
    }))


def cpu_baseline_line(g, x):
    """The reference (oracle/_ref) on the host cores over the same graph (copied
    back from the device), full graph per step, mean of 2 after 1 warmup."""
    from oracle.oracle import Reference, cpu_model, host_threads
    if not Reference.available():
        return None
    src = g.src().cpu().numpy()
    dst = g.dst().cpu().numpy()
    xh = x.cpu().numpy()
    threads = host_threads()
    secs, edges = Reference().bench_spmm(src, dst, N_NODES, N_NODES, xh, threads=threads, rows_limit=0,
                                         warmup=1, repeat=2)
    return {"value": edges / secs / 1e9, "unit": "GEdges/s", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"full graph ({edges} edges), reference spmm<float> sum, "
                      f"{threads} threads over dst-row ranges, mean of 2 after 1 warmup"}


def timed_steps(fn, steps, flush_buf, stream=None):
    """Per-step CUDA-event times (ms) of fn(), L2 flushed by a write larger
    than L2 outside the events before every step, like the headline."""
    fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush_buf.zero_()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def traffic_of(name):
    """Measured DRAM bytes per call from a committed ncu capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get("dram_bytes_per_call")
    except Exception:
        return None


def single_gpu_secondary(gm, L, lib, g, x, cs, plan, flush_buf, steps, hbm):
    """Secondary lines at N = 1, each timed like the headline (per-step events,
    L2 flushed between steps): max + argmax SpMM and CSR build on the same
    graph first, then the segment_matmul lines (tensor-heavy, so they run last
    and cannot leave the SpMM lines at power-capped clocks)."""
    stream = torch.cuda.current_stream()
    sec = {}
    # max + argmax SpMM (the reference's max path, fused; int32 COO-id argmax)
    mo = torch.empty(N_NODES, F, dtype=torch.float32, device=x.device)
    ma = torch.empty(N_NODES, F, dtype=torch.int32, device=x.device)

    def max_step():
        L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), F, None, None,
                            L.GM_MAX, C.c_void_p(mo.data_ptr()), C.c_void_p(ma.data_ptr()),
                            C.c_void_p(stream.cuda_stream)))
    for _ in range(3):
        max_step()
    per = timed_steps(max_step, steps, flush_buf)
    mms = statistics.mean(per)
    mb = spmm_bytes(N_NODES, N_EDGES, F) + N_NODES * F * 4
    sec["max_argmax_spmm"] = {
        "ms": mms, "gedges_s": N_EDGES / mms / 1e6, "per_step_ms": {"min": min(per), "median": statistics.median(per)},
        "roofline": {"bound": "hbm", "achieved": mb / mms / 1e6, "peak": hbm, "unit": "GB/s",
                     "frac": mb / mms / 1e6 / hbm, "traffic": traffic_of("spmm_max_traffic.json"),
                     "algorithmic_bytes_per_call": mb,
                     "bytes_model": "gather model + 4 B int32 argmax per output element"}}
    ma_keep = ma
    del mo
    # CSR build (build_compressed of the CSC: keys = dst, values = src), a fresh
    # build per step (the reference rebuilds it per EdgeIndex, edge_index.cpp:121-136)
    dst, src = g.dst(), g.src()
    ws_bytes = lib.gm_build_compressed_workspace(N_EDGES, N_NODES)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device)
    rp = torch.empty(N_NODES + 1, dtype=torch.int64, device=x.device)
    col = torch.empty(N_EDGES, dtype=torch.int32, device=x.device)
    perm = torch.empty(N_EDGES, dtype=torch.int32, device=x.device)

    def build_step():
        L.check(lib.gm_build_compressed(C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()), N_EDGES, N_NODES,
                                        C.c_void_p(rp.data_ptr()), C.c_void_p(col.data_ptr()),
                                        C.c_void_p(perm.data_ptr()), C.c_void_p(ws.data_ptr()), ws_bytes,
                                        C.c_void_p(stream.cuda_stream)))
    per = timed_steps(build_step, max(3, steps // 3), flush_buf)
    bms = statistics.mean(per)
    bb = 32 * N_EDGES + 8 * (N_NODES + 1)
    csc = g.to_csc()
    same = bool(torch.equal(rp, csc.rowptr) and torch.equal(col, csc.col) and torch.equal(perm, csc.perm))
    sec["csr_build"] = {
        "ms": bms, "gedges_s": N_EDGES / bms / 1e6, "identical_to_cached_csc": same,
        "roofline": {"bound": "hbm", "achieved": bb / bms / 1e6, "peak": hbm, "unit": "GB/s",
                     "frac": bb / bms / 1e6 / hbm, "traffic": traffic_of("csr_build_traffic.json"),
                     "algorithmic_bytes_per_call": bb,
                     "bytes_model": "two-pass stable counting sort: read dst (8E), read dst+src (16E), "
                                    "write col+perm int32 (8E), write rowptr (8(N+1))"}}
    del ws, col, perm
    # backward of the two aggregations (§8f-1), same graph, L2 flushed per step:
    # dw = per-edge dot of the output gradient's destination row with the source
    # row (message_passing.hpp:156-165, CSC order); max backward = argpos scatter
    # + gather_rows adjoint as one gather over the source view (aggregate.hpp:295-308)
    gout = torch.empty_like(x)
    L.check(lib.gm_synth_features(SEED + 7, 0, N_NODES, F, 1, L.GM_F32, C.c_void_p(gout.data_ptr()),
                                  C.c_void_p(stream.cuda_stream)))
    rows = csc.entry_rows()
    dw = torch.empty(N_EDGES, dtype=torch.float32, device=x.device)

    def dw_step():
        L.check(lib.gm_edge_dot_csc(L.GM_F32, C.byref(cs), C.byref(plan), C.c_void_p(rows.data_ptr()),
                                    C.c_void_p(gout.data_ptr()), C.c_void_p(x.data_ptr()), F,
                                    C.c_void_p(dw.data_ptr()), C.c_void_p(stream.cuda_stream)))
    dw_step()
    per = timed_steps(dw_step, max(3, steps // 3), flush_buf)
    dms = statistics.mean(per)
    db = N_EDGES * (F * 4 + 16) + N_NODES * (F * 4 + 8)
    sec["backward_dw"] = {
        "ms": dms, "gedges_s": N_EDGES / dms / 1e6,
        "roofline": {"bound": "hbm", "achieved": db / dms / 1e6, "peak": hbm, "unit": "GB/s",
                     "frac": db / dms / 1e6 / hbm, "algorithmic_bytes_per_call": db,
                     "bytes_model": "per edge: source row gather 4F + col/row/perm/dw 16; per row: gradient row 4F + rowptr 8"}}
    del dw
    view = g.source_view()
    vplan = view.plan(row_bytes=F * 4)
    vcs = view.c_struct()
    dx = torch.empty_like(x)

    def maxbwd_step():
        L.check(lib.gm_spmm_max_backward(C.byref(vcs), C.byref(vplan), L.GM_F32, C.c_void_p(ma_keep.data_ptr()),
                                         C.c_void_p(gout.data_ptr()), F, C.c_void_p(dx.data_ptr()),
                                         C.c_void_p(stream.cuda_stream)))
    maxbwd_step()
    per = timed_steps(maxbwd_step, max(3, steps // 3), flush_buf)
    mbms = statistics.mean(per)
    mbb = N_EDGES * (F * 4 + 8) + N_NODES * (3 * F * 4 + 8)
    sec["backward_max"] = {
        "ms": mbms, "gedges_s": N_EDGES / mbms / 1e6,
        "roofline": {"bound": "hbm", "achieved": mbb / mbms / 1e6, "peak": hbm, "unit": "GB/s",
                     "frac": mbb / mbms / 1e6 / hbm, "algorithmic_bytes_per_call": mbb,
                     "bytes_model": "per source-view entry: destination argmax row 4F + col/eid 8; per row: gradient "
                                    "row 4F (each winner read once), dx row 4F, argmax 4F counted once, rowptr 8"}}
    del dx, gout, ma_keep
    sec["segment_matmul_C3"] = bench_segment_matmul(gm, L, x.device)
    sec["segment_matmul_C3_fp32"] = bench_segment_matmul(gm, L, x.device, fp32=True)
    sec["segment_matmul_F1024"] = bench_segment_matmul(gm, L, x.device, f=1024, rows=500_000)
    sec["segment_matmul_F2048"] = bench_segment_matmul(gm, L, x.device, f=2048, rows=262_144)
    return sec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import paper_2507_16991_b200 as gm
    from paper_2507_16991_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("GM_BENCH_BACKEND", "nccl")  # "gloo": N>1 logic check on one GPU (not a bench)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.current_stream().cuda_stream
    lib = L.lib()

    g, x = make_graph(gm, L, N_NODES, N_EDGES, F, device, stream)
    csc = g.to_csc()
    torch.cuda.synchronize()

    # ---- partition (N > 1): nnz-balanced dst rows, equal-row X shards ----------
    # The timed step at N > 1 is the exchange-overlapped path (BlockedSpmm):
    # the own-shard block aggregates while the CHUNKS async NCCL all-gathers
    # of X are in flight, then each chunk's block continues the rows' sums as
    # it lands. "exact" (one all-gather, then one bit-identical gm_spmm) is
    # timed beside it as a secondary line.
    from paper_2507_16991_b200.dist import BlockedSpmm, allgather_features, chunk_layout, make_shard
    rowptr_h = csc.rowptr.cpu().numpy()
    sh = make_shard(rowptr_h, N_NODES, rank, world)
    r0, r1 = sh.row_begin, sh.row_end
    local_edges = int(rowptr_h[r1] - rowptr_h[r0])
    local_csr = csc if world == 1 else csc.row_slice(r0, r1, local_edges)
    out = torch.empty(N_NODES, F, dtype=torch.float32, device=device)
    x_full = x
    plan = local_csr.plan()
    cs = local_csr.c_struct()
    if world > 1:
        x_full = torch.zeros(sh.shard_rows * world, F, dtype=torch.float32, device=device)
        s_rows, c_rows = chunk_layout(N_NODES, world, CHUNKS)
        lo, hi = rank * s_rows, min((rank + 1) * s_rows, N_NODES)
        x_shard = torch.zeros(CHUNKS * c_rows, F, dtype=torch.float32, device=device)
        x_shard[: max(0, hi - lo)].copy_(x[lo:hi])
        blocked = BlockedSpmm(local_csr, N_NODES, rank, world, CHUNKS)
        out_local = out[r0:r1]

    def step_exact():
        if world > 1:
            allgather_features(x_shard[: sh.shard_rows], sh, out=x_full)
        L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x_full.data_ptr()), F, None,
                            None, L.GM_SUM, C.c_void_p(out[r0:].data_ptr()), None,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def step():
        if world > 1:
            blocked(x_shard, "sum", out=out_local)
        else:
            step_exact()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # L2 (126 MB) is flushed between timed steps by a 256 MB write outside the
    # events, so no step sees rows a previous step left resident.
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        for i in range(args.steps):
            flush_buf.zero_()
            evs[i][0].record()
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    per_step = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(per_step)
    if dist:
        t = torch.tensor([total_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    value = N_EDGES / (ms * 1e-3) / 1e9

    hbm, bf16_peak, peak_kind = peaks()
    # roofline of the dominant launch (one gm_spmm call = light + concurrent hub kernel)
    call_ms = statistics.mean(per_step) if world == 1 else None
    roof = None
    if world == 1:
        b = spmm_bytes(N_NODES, N_EDGES, F)
        ach = b / (call_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "spmm_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_call")
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic, "peak_kind": peak_kind, "algorithmic_bytes_per_call": b,
                "unit_of_launch": "one gm_spmm call (warp-window kernel + concurrent hub-row kernel)"}

    # ---- e2e through the public C-ABI with host buffers (N = 1) -----------------
    # Every step copies its input X (pinned host -> device), runs gm_spmm and
    # reads its output back (device -> pinned host). Steps are pipelined on
    # three streams with double-buffered device X/out: H2D of step i+1 and D2H
    # of step i-1 overlap the SpMM of step i (PCIe is full duplex). The serial
    # (unpipelined) figure is reported beside it.
    e2e = None
    if world == 1:
        xh = torch.empty(N_NODES, F, dtype=torch.float32).pin_memory()
        ohs = [torch.empty(N_NODES, F, dtype=torch.float32).pin_memory() for _ in range(2)]
        xh.copy_(x.cpu())
        xds = [torch.empty_like(x) for _ in range(2)]
        outs = [torch.empty_like(x) for _ in range(2)]
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        e2e_steps = max(4, min(args.steps, 10))

        def spmm_on(xd, od, stream):
            L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(xd.data_ptr()), F, None,
                                None, L.GM_SUM, C.c_void_p(od.data_ptr()), None, C.c_void_p(stream.cuda_stream)))

        def run_pipelined(steps):
            h2d = [torch.cuda.Event() for _ in range(2)]
            cmp = [torch.cuda.Event() for _ in range(2)]
            d2h = [torch.cuda.Event() for _ in range(2)]
            for i in range(steps):
                b = i % 2
                if i >= 2:
                    s_in.wait_event(cmp[b])     # xds[b] free again
                with torch.cuda.stream(s_in):
                    xds[b].copy_(xh, non_blocking=True)
                    h2d[b].record(s_in)
                s_cmp.wait_event(h2d[b])
                if i >= 2:
                    s_cmp.wait_event(d2h[b])    # outs[b] read back already
                spmm_on(xds[b], outs[b], s_cmp)
                cmp[b].record(s_cmp)
                s_out.wait_event(cmp[b])
                with torch.cuda.stream(s_out):
                    ohs[b].copy_(outs[b], non_blocking=True)
                    d2h[b].record(s_out)

        run_pipelined(2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = torch.cuda.Event(enable_timing=True)
        bev = torch.cuda.Event(enable_timing=True)
        a.record(s_in)
        run_pipelined(e2e_steps)
        s_in.wait_stream(s_out)
        bev.record(s_in)
        torch.cuda.synchronize()
        ems = a.elapsed_time(bev) / e2e_steps
        wall_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps

        # serial reference point: copy in, aggregate, copy out, one step at a time
        a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a2.record()
        for _ in range(3):
            xds[0].copy_(xh, non_blocking=True)
            spmm_on(xds[0], outs[0], cur)
            ohs[0].copy_(outs[0], non_blocking=True)
        b2.record()
        torch.cuda.synchronize()
        sms = a2.elapsed_time(b2) / 3
        assert torch.equal(ohs[0], ohs[1]), "pipelined and serial e2e outputs differ"
        e2e = {"value": N_EDGES / (ems * 1e-3) / 1e9, "unit": "GEdges/s",
               "h2d_bytes_per_step": N_NODES * F * 4, "d2h_bytes_per_step": N_NODES * F * 4,
               "ms_per_step": ems, "wall_ms_per_step": wall_ms, "mode": "3-stream pipelined across steps",
               "serial_value": N_EDGES / (sms * 1e-3) / 1e9, "serial_ms_per_step": sms}

    secondary = None

    def multi_gpu_secondary():
        # exact mode: one all-gather, then one bit-identical gm_spmm per rank
        for _ in range(2):
            step_exact()
        torch.cuda.synchronize()
        dist.barrier()
        a, bev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            step_exact()
        bev.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(bev) / 5], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        exact_ms = float(t.item())
        # numerics check at N > 1: overlap-mode rows vs the exact (1-GPU-identical) rows
        blk_out = torch.empty_like(out_local)
        blocked(x_shard, "sum", out=blk_out)
        torch.cuda.synchronize()
        diff = (blk_out - out_local).abs().max()
        ref_mag = out_local.abs().max()
        chk = torch.stack([diff, ref_mag])
        dist.all_reduce(chk, op=dist.ReduceOp.MAX)
        # halo-only exchange: one all_to_all of the referenced remote rows
        from paper_2507_16991_b200.dist import HaloSpmm, exchange_need_lists, halo_need
        need = halo_need(local_csr, N_NODES, rank, world)
        halo = HaloSpmm(local_csr, N_NODES, rank, world, need, exchange_need_lists(need))
        xs = x_shard[: sh.shard_rows]
        for _ in range(2):
            halo(xs, "sum", out=out_local)
        torch.cuda.synchronize()
        dist.barrier()
        a.record()
        for _ in range(5):
            halo(xs, "sum", out=out_local)
        bev.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(bev) / 5, float(halo.halo_rows())], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return {"exact_mode_spmm": {"ms": exact_ms, "gedges_s": N_EDGES / exact_ms / 1e6,
                                         "numerics": "bit-identical to 1 GPU"},
                     "halo_mode_spmm": {"ms": float(t[0]), "gedges_s": N_EDGES / float(t[0]) / 1e6,
                                        "max_halo_rows": int(t[1]), "halo_frac_of_remote_rows":
                                        float(t[1]) / (N_NODES - sh.shard_rows)},
                     "overlap_mode_numerics": "sum continued across 1+CHUNKS source blocks (fp32 tolerance)",
                "overlap_vs_exact_max_abs_diff": float(chk[0]), "exact_max_abs": float(chk[1]),
                     "block_nnz": blocked.block_nnz(),
                     "segment_matmul_C3": bench_segment_matmul(gm, L, device, rank=rank, world=world, dist=dist),
                     "segment_matmul_F1024": bench_segment_matmul(gm, L, device, f=1024, rows=500_000, rank=rank,
                                                                  world=world, dist=dist)}
    if world > 1 and not args.no_secondary:
        try:  # reported, never substituted for the headline
            secondary = multi_gpu_secondary()
        except Exception as exc:  # noqa: BLE001
            secondary = {"error": str(exc)[:300]}
    if world == 1 and not args.no_secondary:
        secondary = single_gpu_secondary(gm, L, lib, g, x, cs, plan, flush_buf, args.steps, hbm)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(g, x)
        except Exception as exc:
            cpu = {"error": str(exc)[:200]}

    launches_per_step = 1 + (1 if plan.num_heavy > 0 else 0)
    if world > 1:
        launches_per_step = sum(1 + (1 if v.plan().num_heavy > 0 else 0) for v in blocked.blocks)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GEdges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(world),
            "plan": {"l2_hot_mb": int(plan.l2_hot_bytes >> 20), "heavy_rows": int(plan.num_heavy)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(), "secondary": secondary,
            "per_step_ms": {"min": min(per_step), "median": statistics.median(per_step), "max": max(per_step)},
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
