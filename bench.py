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


def workload_config(world: int, mode: str = "push") -> dict:
    """The `config` both arms print (same workload, same keys)."""
    par = f"dst-row partition x{world}"
    if world > 1:
        par += (" (each rank builds its CSC rows from its own COO chunk); " + (
            "push mode: the SpMM epilogue stores finished rows into the referencing peers' next-layer X "
            "over NVLink P2P, one 1-element all_reduce per step" if mode == "push" else
            f"{CHUNKS} chunked async NCCL all-gathers of X overlapped with source-blocked aggregation"))
    return {"workload": "ogbn-products-shaped power-law graph (configs[3]), full-graph sum SpMM",
            "nodes": N_NODES, "edges": N_EDGES, "feats": F, "graph": "Chung-Lu alpha=0.5",
            "seed": hex(SEED), "parallelism": par, "mode": mode if world > 1 else "single GPU",
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
                     "traffic": traffic_of("backward_dw_traffic.json"),
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
                     "traffic": traffic_of("backward_max_traffic.json"),
                     "bytes_model": "per source-view entry: destination argmax row 4F + col/eid 8; per row: gradient "
                                    "row 4F (each winner read once), dx row 4F, argmax 4F counted once, rowptr 8"}}
    del dx, gout, ma_keep
    sec["segment_matmul_C3"] = bench_segment_matmul(gm, L, x.device)
    sec["segment_matmul_C3_fp32"] = bench_segment_matmul(gm, L, x.device, fp32=True)
    sec["segment_matmul_F1024"] = bench_segment_matmul(gm, L, x.device, f=1024, rows=500_000)
    sec["segment_matmul_F2048"] = bench_segment_matmul(gm, L, x.device, f=2048, rows=262_144)
    return sec


def main_multi(args, world, rank, local):
    """N > 1 (one process per GPU): every rank generates only its chunk of the
    COO edge list and builds its CSC row slice with the distributed
    build_compressed (dist.build_local_csc: degree all-reduce, nnz cuts, one
    edge all_to_all, local stable build). Headline step (GM_BENCH_MODE=push,
    default): the push-mode SpMM — every rank aggregates its destination rows
    from its replica of X and its epilogue stores each finished row into the
    peers' next-layer replicas over NVLink P2P (halo masks: only to peers that
    reference the row); a one-element all_reduce orders the next reads. The
    output of step s is the input of step s+1 (ping-pong replicas), i.e. the
    steady state of a multi-layer model. GM_BENCH_MODE=blocked: CHUNKS async
    all-gathers of X overlapped with source-blocked aggregation. The other
    modes (exact, blocked, halo, C5-shaped bf16) are secondary lines."""
    import torch.distributed as dist

    import paper_2507_16991_b200 as gm
    from paper_2507_16991_b200 import _lib as L
    from paper_2507_16991_b200 import dist as gd

    device = torch.device("cuda", local)
    backend = os.environ.get("GM_BENCH_BACKEND", "nccl")  # "gloo": N>1 logic check on one GPU (not a bench)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group(backend)
    stream = torch.cuda.current_stream().cuda_stream
    lib = L.lib()
    hbm, bf16_peak, peak_kind = peaks()

    def local_graph(n, e, seed):
        e0, e1 = rank * e // world, (rank + 1) * e // world
        src = torch.empty(e1 - e0, dtype=torch.int64, device=device)
        dst = torch.empty(e1 - e0, dtype=torch.int64, device=device)
        L.check(lib.gm_synth_edges(1, seed, e0, e1 - e0, n, n, src.data_ptr(), dst.data_ptr(), stream))
        cuts, rows = gd.build_local_csc(src, dst, e0, n, rank, world)
        return cuts, rows

    def maxed(vals):
        t = torch.tensor([float(v) for v in vals], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def timed(step, steps, warmup, flush_buf):
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            flush_buf.zero_()
            evs[i][0].record()
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
        dist.barrier()
        per = [a.elapsed_time(b) for a, b in evs]
        return maxed([sum(per) / steps])[0], per

    cuts, rows = local_graph(N_NODES, N_EDGES, SEED)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    local_edges = rows.num_entries()
    x = torch.empty(N_NODES, F, dtype=torch.float32, device=device)  # replica: identical on every rank
    L.check(lib.gm_synth_features(SEED, 0, N_NODES, F, 0, L.GM_F32, x.data_ptr(), stream))
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    mode = os.environ.get("GM_BENCH_MODE", "push")
    push_note = None
    mask = None
    if mode == "push":
        try:
            xb = torch.empty_like(x)
            ptr_b, bases_b = gd.open_peer_buffers(xb)
            mask = gd.push_masks(rows, N_NODES, r0, r1, rank, world)
            op = gd.PushSpmm(rows, r0, r1, rank, world, mask)
            one = torch.ones(1, device=device)

            def step():
                # one layer: aggregate this rank's rows of X, push them into every
                # referencing peer's next-layer input (xb), then order the reads
                op(x, xb, ptr_b)
                dist.all_reduce(one)
        except Exception as exc:  # noqa: BLE001 - no P2P mapping here: the overlap mode is the headline
            push_note = f"push mode unavailable ({str(exc)[:160]}); blocked mode timed instead"
            mode = "blocked"
    s_rows, c_rows = gd.chunk_layout(N_NODES, world, CHUNKS)
    lo, hi = rank * s_rows, min((rank + 1) * s_rows, N_NODES)
    x_shard = torch.zeros(CHUNKS * c_rows, F, dtype=torch.float32, device=device)
    x_shard[: max(0, hi - lo)].copy_(x[lo:hi])
    blocked = gd.BlockedSpmm(rows, N_NODES, rank, world, CHUNKS)
    out_local = torch.empty(r1 - r0, F, dtype=torch.float32, device=device)
    if mode == "blocked":
        def step():
            blocked(x_shard, "sum", out=out_local)

    with ClockSampler(local) as clk:
        ms, per_step = timed(step, args.steps, args.warmup, flush_buf)
    value = N_EDGES / (ms * 1e-3) / 1e9

    # roofline at N: the slowest rank's local gather-model bytes against its
    # HBM, plus the exchange each step needs (NVLink 5: 900 GB/s per direction)
    lb = spmm_bytes(r1 - r0, local_edges, F)
    if mode == "push":
        peers_per_row = (torch.bitwise_and(mask.view(-1, 1), torch.tensor([1 << j for j in range(world - 1)],
                         dtype=torch.int32, device=device)) != 0).sum() if mask is not None else (r1 - r0) * (world - 1)
        xbytes = int(peers_per_row) * F * 4
        xkind = "push: rows stored by the SpMM epilogue into referencing peers (NVLink P2P)"
    else:
        xbytes = (world - 1) * s_rows * F * 4
        xkind = "chunked all-gather of X shards (received per rank)"
    lb_max, xb_max = maxed([lb, xbytes])
    nvlink = 900.0
    roof = {"bound": "hbm", "achieved": lb_max / ms / 1e6, "peak": hbm, "unit": "GB/s",
            "frac": lb_max / ms / 1e6 / hbm, "traffic": None, "peak_kind": peak_kind,
            "algorithmic_bytes_per_call": lb_max,
            "unit_of_launch": "the slowest rank's SpMM over its destination rows (gather model)",
            "exchange": {"mode": xkind, "bytes_per_rank_max": xb_max, "nvlink_gbs": nvlink,
                         "nvlink_floor_ms": xb_max / nvlink / 1e6, "hbm_floor_ms": lb_max / hbm / 1e6,
                         "step_floor_ms": max(xb_max / nvlink / 1e6, lb_max / hbm / 1e6)}}

    push_check = None
    if mode == "push":
        # end-to-end numerics at N: the rows this rank reads next (its own +
        # every source it references) must equal the exact (all-gather +
        # single-GPU kernel) output of their owners, bit for bit
        s_rows_ = -(-N_NODES // world)
        sh = gd.Shard(rank, world, r0, r1, s_rows_)
        x_full = torch.empty(s_rows_ * world, F, dtype=torch.float32, device=device)
        gd.allgather_features(x_shard[:s_rows_], sh, out=x_full)
        ex = torch.empty(r1 - r0, F, dtype=torch.float32, device=device)
        cs_ = rows.c_struct()
        L.check(lib.gm_spmm(C.byref(cs_), C.byref(rows.plan(F * 4)), L.GM_F32, C.c_void_p(x_full.data_ptr()), F, None,
                            None, L.GM_SUM, C.c_void_p(ex.data_ptr()), None, C.c_void_p(stream)))
        rmax = int(maxed([r1 - r0])[0])
        pad = torch.zeros(rmax, F, dtype=torch.float32, device=device)
        pad[: r1 - r0].copy_(ex)
        allx = torch.empty(world * rmax, F, dtype=torch.float32, device=device)
        dist.all_gather_into_tensor(allx, pad)
        full = torch.cat([allx[q * rmax:q * rmax + int(cuts[q + 1] - cuts[q])] for q in range(world)])
        mark = torch.empty(N_NODES, dtype=torch.uint8, device=device)
        L.check(lib.gm_mark_columns(C.byref(cs_), C.c_void_p(mark.data_ptr()), C.c_void_p(stream)))
        need = mark != 0
        need[r0:r1] = True
        bad = int(maxed([float((xb[need] != full[need]).any(dim=1).sum())])[0])
        push_check = {"rows_checked_per_rank": int(need.sum()), "mismatched_rows_max_over_ranks": bad,
                      "reference": "exact mode (all-gather + single-GPU gm_spmm)"}
        del x_full, allx, full
        gd.close_peer_buffers(bases_b)
    secondary = None
    if not args.no_secondary:
        try:
            secondary = multi_secondary(args, gm, L, gd, dist, lib, device, rank, world, rows, cuts, x, x_shard,
                                        blocked, out_local, flush_buf, timed, maxed, local_graph, mode)
        except Exception as exc:  # noqa: BLE001 - reported, never substituted for the headline
            secondary = {"error": str(exc)[:300]}
    plan = rows.plan(F * 4)
    launches = 1 + (1 if plan.num_heavy > 0 else 0)
    if mode == "blocked":
        launches = sum(1 + (1 if v.plan(F * 4).num_heavy > 0 else 0) for v in blocked.blocks)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "GEdges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(world, mode), **({"note": push_note} if push_note else {})),
            "push_numerics": push_check,
            "roofline": roof, "cpu_baseline": None, "e2e": None, "gpu_launches": launches * args.steps,
            "clocks": clk.summary(), "secondary": secondary,
            "per_step_ms": {"min": min(per_step), "median": statistics.median(per_step), "max": max(per_step), "mean": statistics.mean(per_step), "std": statistics.pstdev(per_step)},
        }))
    dist.destroy_process_group()


def multi_secondary(args, gm, L, gd, dist, lib, device, rank, world, rows, cuts, x, x_shard, blocked, out_local,
                    flush_buf, timed, maxed, local_graph, mode):
    """Secondary lines at N > 1, each timed like the headline (max over ranks)."""
    sec = {}
    steps = max(3, args.steps // 3)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    stream = torch.cuda.current_stream().cuda_stream
    s_rows = -(-N_NODES // world)
    sh = gd.Shard(rank, world, r0, r1, s_rows)
    cs = rows.c_struct()
    plan = rows.plan(F * 4)
    x_full = torch.empty(s_rows * world, F, dtype=torch.float32, device=device)

    def step_exact():
        gd.allgather_features(x_shard[:s_rows], sh, out=x_full)
        L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x_full.data_ptr()), F, None, None,
                            L.GM_SUM, C.c_void_p(out_local.data_ptr()), None, C.c_void_p(stream)))
    ms, _ = timed(step_exact, steps, 2, flush_buf)
    sec["exact_mode_spmm"] = {"ms": ms, "gedges_s": N_EDGES / ms / 1e6, "numerics": "bit-identical to 1 GPU"}
    exact = out_local.clone()
    if mode != "blocked":
        ms, _ = timed(lambda: blocked(x_shard, "sum", out=out_local), steps, 2, flush_buf)
        sec["blocked_mode_spmm"] = {"ms": ms, "gedges_s": N_EDGES / ms / 1e6, "chunks": CHUNKS,
                                    "numerics": "sums continued across 1+CHUNKS source blocks (fp32 tolerance)"}
    blocked(x_shard, "sum", out=out_local)
    torch.cuda.synchronize()
    d, m = maxed([float((out_local - exact).abs().max()), float(exact.abs().max())])
    sec["blocked_vs_exact_max_abs_diff"] = d
    sec["exact_max_abs"] = m
    need = gd.halo_need(rows, N_NODES, rank, world)
    halo = gd.HaloSpmm(rows, N_NODES, rank, world, need, gd.exchange_need_lists(need))
    xs = x_shard[:s_rows]
    ms, _ = timed(lambda: halo(xs, "sum", out=out_local), steps, 2, flush_buf)
    hr = maxed([float(halo.halo_rows())])[0]
    sec["halo_mode_spmm"] = {"ms": ms, "gedges_s": N_EDGES / ms / 1e6, "max_halo_rows": int(hr),
                             "halo_frac_of_remote_rows": hr / (N_NODES - s_rows)}
    sec["block_nnz"] = blocked.block_nnz()
    # C5-shaped (ogbn-papers100M: F = 128 bf16, Chung-Lu alpha 0.5) at 1/16 of its size per the
    # whole job, blocked mode with the fp32 carry (bf16 sums rounded once per row)
    n5, e5, f5 = 111_059_956 // 16, 1_615_685_872 // 16, 128
    cuts5, rows5 = local_graph(n5, e5, SEED + 5)
    a5, b5 = int(cuts5[rank]), int(cuts5[rank + 1])
    s5, c5 = gd.chunk_layout(n5, world, CHUNKS)
    x5 = torch.empty(min(s5, n5 - rank * s5), f5, dtype=torch.bfloat16, device=device)
    L.check(lib.gm_synth_features(SEED + 5, rank * s5, x5.shape[0], f5, 0, L.GM_BF16, x5.data_ptr(), stream))
    xs5 = torch.zeros(CHUNKS * c5, f5, dtype=torch.bfloat16, device=device)
    xs5[: x5.shape[0]].copy_(x5)
    del x5
    blk5 = gd.BlockedSpmm(rows5, n5, rank, world, CHUNKS)
    o5 = torch.empty(b5 - a5, f5, dtype=torch.bfloat16, device=device)
    ms, _ = timed(lambda: blk5(xs5, "sum", out=o5), steps, 2, flush_buf)
    hbm = peaks()[0]
    lb5 = maxed([spmm_bytes(b5 - a5, rows5.num_entries(), f5, esz=2)])[0]
    sec["c5_shape_bf16_blocked"] = {
        "nodes": n5, "edges": e5, "feats": f5, "ms": ms, "gedges_s": e5 / ms / 1e6,
        "roofline": {"bound": "hbm", "achieved": lb5 / ms / 1e6, "peak": hbm, "frac": lb5 / ms / 1e6 / hbm},
        "numerics": "bf16 sums carried in fp32 across the 1+CHUNKS blocks, one rounding per row"}
    del blk5, xs5, rows5
    sec["segment_matmul_C3"] = bench_segment_matmul(gm, L, device, rank=rank, world=world, dist=dist)
    sec["segment_matmul_F1024"] = bench_segment_matmul(gm, L, device, f=1024, rows=500_000, rank=rank, world=world,
                                                       dist=dist)
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
    if world > 1:
        main_multi(args, world, rank, local)
        return
    device = torch.device("cuda", local)
    stream = torch.cuda.current_stream().cuda_stream
    lib = L.lib()

    g, x = make_graph(gm, L, N_NODES, N_EDGES, F, device, stream)
    csc = g.to_csc()
    torch.cuda.synchronize()
    out = torch.empty(N_NODES, F, dtype=torch.float32, device=device)
    plan = csc.plan()
    cs = csc.c_struct()

    def step():
        L.check(lib.gm_spmm(C.byref(cs), C.byref(plan), L.GM_F32, C.c_void_p(x.data_ptr()), F, None,
                            None, L.GM_SUM, C.c_void_p(out.data_ptr()), None,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # L2 (126 MB) is flushed between timed steps by a 256 MB write outside the
    # events, so no step sees rows a previous step left resident.
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush_buf.zero_()
            evs[i][0].record()
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
    per_step = [a.elapsed_time(b) for a, b in evs]
    ms = sum(per_step) / args.steps
    value = N_EDGES / (ms * 1e-3) / 1e9

    hbm, bf16_peak, peak_kind = peaks()
    # roofline of the dominant launch (one gm_spmm call = light + concurrent hub kernel)
    call_ms = statistics.mean(per_step)
    roof = None
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
    xh = torch.empty(N_NODES, F, dtype=torch.float32).pin_memory()
    ohs = [torch.empty(N_NODES, F, dtype=torch.float32).pin_memory() for _ in range(2)]
    xh.copy_(x.cpu())
    xds = [torch.empty_like(x) for _ in range(2)]
    outs = [torch.empty_like(x) for _ in range(2)]
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    # the same K steps as the device-timed region (the pipeline's fill and
    # drain — one unoverlapped copy each way — amortise over the K steps)
    e2e_steps = max(4, args.steps)

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
    if not args.no_secondary:
        secondary = single_gpu_secondary(gm, L, lib, g, x, cs, plan, flush_buf, args.steps, hbm)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(g, x)
        except Exception as exc:
            cpu = {"error": str(exc)[:200]}

    launches_per_step = 1 + (1 if plan.num_heavy > 0 else 0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GEdges/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(1),
            "plan": {"l2_hot_mb": int(plan.l2_hot_bytes >> 20), "heavy_rows": int(plan.num_heavy)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(), "secondary": secondary,
            "per_step_ms": {"min": min(per_step), "median": statistics.median(per_step), "max": max(per_step), "mean": statistics.mean(per_step), "std": statistics.pstdev(per_step)},
        }
        print(json.dumps(line))


if __name__ == "__main__":
    main()
