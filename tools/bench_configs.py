"""Throughput of every BASELINE.json config on one B200 (CUDA events, L2
flushed between timed calls, warmup 3). Prints one JSON object per config.

  C1 Cora-shaped 2-layer GCN forward (fp32, 1433 -> 16 -> 16 -> head 7)
  C2 Reddit-shaped mean SpMM (F=602 fp32)
  C3 OGB-MAG segment_matmul (K=N=128 bf16)  [+ per-edge-type mean SpMM at F=128]
  C4 ogbn-products sum / max+argmax SpMM (F=100 fp32)
  C5 ogbn-papers100M sum SpMM (F=128 bf16)
"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_16991_b200 as gm  # noqa: E402
from paper_2507_16991_b200 import _lib as L  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM = PEAKS["hbm_gbs"]
SEED = 0x67726170686D696C
FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


def graph(kind, n, e, seed=SEED):
    s = torch.empty(e, dtype=torch.int64, device="cuda")
    d = torch.empty(e, dtype=torch.int64, device="cuda")
    L.check(L.lib().gm_synth_edges(kind, seed, 0, e, n, n, s.data_ptr(), d.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
    return gm.EdgeIndex(s, d, n, n)


def feats(n, f, dtype):
    x = torch.empty(n, f, dtype=dtype, device="cuda")
    code = {torch.float32: L.GM_F32, torch.bfloat16: L.GM_BF16}[dtype]
    L.check(L.lib().gm_synth_features(SEED, 0, n, f, 0, code, x.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return x


def spmm_line(name, kind, n, e, f, dtype, reduce):
    g = graph(kind, n, e)
    x = feats(n, f, dtype)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    csc = g.to_csc()
    t1.record()
    torch.cuda.synchronize()
    build_ms = t0.elapsed_time(t1)
    csc.plan()
    if reduce in ("max", "min"):
        ms = timed(lambda: gm.neighbor_aggregate(g, x, reduce, return_argmax=True))
    else:
        ms = timed(lambda: gm.spmm(g, x, None, reduce))
    s = x.element_size()
    byts = e * (f * s + 4) + n * (8 + f * s) + (n * f * 4 if reduce in ("max", "min") else 0)
    r = {"config": name, "reduce": reduce, "dtype": str(dtype).split(".")[-1], "nodes": n, "edges": e, "feats": f,
         "ms": ms, "gedges_s": e / ms / 1e6, "algo_gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / HBM,
         "csc_build_ms": build_ms, "heavy_rows": int(csc.plan().num_heavy)}
    if os.environ.get("GM_AB_HASH"):  # bit hash of the output (same-box A/B of layout knobs)
        o = gm.neighbor_aggregate(g, x, reduce, return_argmax=True)[0] if reduce in ("max", "min") else gm.spmm(g, x, None, reduce)
        bits = o.contiguous().view(torch.int32 if o.element_size() == 4 else torch.int16).flatten()
        acc, step = 0, 1 << 26  # chunked: a C5 output is 14 G elements
        for c0 in range(0, bits.numel(), step):
            b = bits[c0:c0 + step].to(torch.int64)
            idx = torch.arange(c0 + 1, c0 + 1 + b.numel(), device=b.device, dtype=torch.int64)
            acc += int((b * idx % 1000003).sum().item())
        r["out_hash"] = acc
    print(json.dumps(r), flush=True)
    del g, x, csc
    torch.cuda.empty_cache()
    return r


def cora():
    n, e = 2708, 10556
    g = graph(0, n, e)
    torch.manual_seed(0)
    h = torch.randn(n, 1433, device="cuda")
    w1, w2, wh = (torch.randn(1433, 16, device="cuda") / 38, torch.randn(16, 16, device="cuda") / 4,
                  torch.randn(16, 7, device="cuda") / 4)
    b1, b2, bh = torch.zeros(16, device="cuda"), torch.zeros(16, device="cuda"), torch.zeros(7, device="cuda")

    def fwd():
        z = torch.relu(gm.gcn_layer(g, h, w1, b1))
        z = gm.gcn_layer(g, z, w2, b2)
        return z @ wh + bh

    ms = timed(fwd, reps=50)
    # the same forward captured once into a CUDA graph and replayed (launch-bound config)
    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        static_out = fwd()
    ref = fwd()
    cg.replay()
    torch.cuda.synchronize()
    assert torch.equal(static_out, ref), "graph replay differs from eager"
    gms = timed(cg.replay, reps=200)
    r = {"config": "C1 cora 2-layer GCN forward", "ms": ms, "graph_replay_ms": gms, "nodes": n, "edges": e,
         "feats": 1433, "note": "launch-bound (2 transforms + 2 fused GCN SpMMs + head); parity config"}
    print(json.dumps(r), flush=True)


def mag_gemm():
    ptr = [0, 736_389, 1_871_038, 1_879_778, 1_939_743]
    x = torch.randn(ptr[-1], 128, device="cuda").to(torch.bfloat16)
    w = (torch.randn(4, 128, 128, device="cuda") / 11).to(torch.bfloat16)
    ms = timed(lambda: gm.segment_matmul(x, ptr, w), reps=20)
    flops = 2.0 * ptr[-1] * 128 * 128
    byts = 2.0 * ptr[-1] * 256 + 4 * 128 * 128 * 2
    r = {"config": "C3 ogb-mag segment_matmul", "ms": ms, "tflops": flops / ms / 1e9,
         "algo_gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / HBM,
         "frac_tensor": flops / ms / 1e9 / PEAKS["bf16_tflops"]}
    print(json.dumps(r), flush=True)
    # the reference's own dtype: fp32 operands, fp32-accurate 3-piece split path
    xf, wf = x.float(), w.float()
    ms = timed(lambda: gm.segment_matmul(xf, ptr, wf), reps=20)
    byts = 4.0 * ptr[-1] * 256 + 4 * 128 * 128 * 4
    r = {"config": "C3 ogb-mag segment_matmul fp32 operands (fp32-accurate split)", "ms": ms,
         "tflops": flops / ms / 1e9, "algo_gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / HBM}
    print(json.dumps(r), flush=True)


def products_backward():
    """C4 backward of a weighted sum SpMM: dx (transposed product over the
    CSR-by-source cache) and dw (per-edge dot), message_passing.hpp:119-166."""
    n, e, f = 2_449_029, 61_859_140, 100
    g = graph(1, n, e)
    x = feats(n, f, torch.float32)
    w = torch.rand(e, device="cuda") + 0.5
    gout = feats(n, f, torch.float32)
    g.to_csr().plan(row_bytes=f * 4)
    dx_ms = timed(lambda: gm.spmm_backward(g, x, None, "sum", gout), reps=5)
    wfwd_ms = timed(lambda: gm.spmm(g, x, w, "sum"), reps=5)
    src, dst = g.src(), g.dst()
    dw = torch.empty(e, device="cuda")
    dot_ms = timed(lambda: L.check(L.lib().gm_edge_dot(L.GM_F32, src.data_ptr(), dst.data_ptr(), e, gout.data_ptr(),
                                                       x.data_ptr(), f, dw.data_ptr(),
                                                       torch.cuda.current_stream().cuda_stream)), reps=5)
    full_ms = timed(lambda: gm.spmm_backward(g, x, w, "sum", gout), reps=5)
    csc = g.to_csc()
    cs = csc.c_struct()
    er = csc.entry_rows()
    import ctypes as _C
    dot_csc_ms = timed(lambda: L.check(L.lib().gm_edge_dot_csc(L.GM_F32, _C.byref(cs), _C.byref(csc.plan()), er.data_ptr(), gout.data_ptr(),
                                                               x.data_ptr(), f, dw.data_ptr(),
                                                               torch.cuda.current_stream().cuda_stream)), reps=5)
    r = {"config": "C4 backward (sum)", "edge_dot_csc_ms": dot_csc_ms, "dx_ms": dx_ms, "dx_gedges_s": e / dx_ms / 1e6, "dx_and_dw_ms": full_ms,
         "weighted_fwd_ms": wfwd_ms, "edge_dot_ms": dot_ms}
    print(json.dumps(r), flush=True)


def mag_layer():
    """C3 end-to-end RGCN-shaped hetero SAGE layer (bf16 weights -> bf16 GEMMs)."""
    from paper_2507_16991_b200.hetero import hetero_sage_layer
    counts = {"paper": 736_389, "author": 1_134_649, "institution": 8_740, "field_of_study": 59_965}
    rels = [("author", "writes", "paper", 7_145_660), ("author", "affiliated_with", "institution", 1_043_998),
            ("paper", "cites", "paper", 5_416_271), ("paper", "has_topic", "field_of_study", 7_505_078)]
    torch.manual_seed(0)
    h = {t: torch.randn(c, 128, device="cuda") for t, c in counts.items()}
    edges, wn = {}, {}
    for i, (s_t, r, d_t, m) in enumerate(rels):
        src = torch.empty(m, dtype=torch.int64, device="cuda")
        dst = torch.empty(m, dtype=torch.int64, device="cuda")
        L.check(L.lib().gm_synth_edges(0, SEED + i, 0, m, counts[s_t], counts[d_t], src.data_ptr(), dst.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream))
        edges[(s_t, r, d_t)] = gm.EdgeIndex(src, dst, counts[s_t], counts[d_t])
        wn[(s_t, r, d_t)] = (torch.randn(128, 128, device="cuda") / 11).to(torch.bfloat16)
    ws = {t: (torch.randn(128, 128, device="cuda") / 11).to(torch.bfloat16) for t in counts}
    b = {t: torch.zeros(128, device="cuda") for t in counts}
    ms = timed(lambda: hetero_sage_layer(edges, h, wn, ws, b), reps=10)
    e_tot = sum(m for *_, m in rels)
    r = {"config": "C3 hetero SAGE layer (4 relations mean SpMM + 2 grouped GEMMs + combine, bf16 W)", "ms": ms,
         "edges": e_tot, "nodes": sum(counts.values())}
    print(json.dumps(r), flush=True)
    # the reference's dtype throughout: fp32 weights -> fp32-accurate fused-split GEMMs
    wn32 = {k: v.float() for k, v in wn.items()}
    ws32 = {k: v.float() for k, v in ws.items()}
    ms = timed(lambda: hetero_sage_layer(edges, h, wn32, ws32, b), reps=10)
    r = {"config": "C3 hetero SAGE layer, fp32 W (fp32-accurate GEMMs)", "ms": ms,
         "edges": e_tot, "nodes": sum(counts.values())}
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    if "C1" in which:
        cora()
    if "C3" in which:
        mag_gemm()
        spmm_line("C3 ogb-mag per-relation mean SpMM (writes, 1.13M->0.74M)", 0, 1_134_649, 7_145_660, 128,
                  torch.float32, "mean")
    if "C4" in which:
        spmm_line("C4 ogbn-products", 1, 2_449_029, 61_859_140, 100, torch.float32, "sum")
        spmm_line("C4 ogbn-products", 1, 2_449_029, 61_859_140, 100, torch.float32, "max")
    if "C2" in which:
        spmm_line("C2 reddit", 1, 232_965, 114_615_892, 602, torch.float32, "mean")
    if "C2X" in which:
        spmm_line("C2 reddit", 1, 232_965, 114_615_892, 602, torch.float32, "max")
    if "C4B" in which:
        products_backward()
    if "C3L" in which:
        mag_layer()
    if "C5" in which:
        spmm_line("C5 ogbn-papers100M (1 GPU)", 1, 111_059_956, 1_615_685_872, 128, torch.bfloat16, "sum")
