"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the container that has /root/reference:
    make -C oracle ref && python tests/make_golden.py
    python tests/make_golden.py --dataset      (reference-written dataset dirs)

Every expected output below is produced by the reference's own code
(build_compressed, spmm, the max path + backward argpos, aggregate, the GCN
branch, grouped_matmul) through oracle/ref_capi.cpp. Inputs of the "ref_*"
cases reproduce the reference tests' exact inputs via tests/refrng.py
(test_stream salts from test_*.cpp); the "syn_*" cases are larger synthetic
graphs (stored in full) that exercise odd widths, hubs (> the 1024-edge heavy
threshold and > the 4096-entry big-row sort), ties and bf16 rounding.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.oracle import Reference  # noqa: E402
import refrng  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def bf16_round(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


def csr_fixtures(ref: Reference) -> dict:
    d = {}
    cases = {
        "diamond": (np.array([0, 1, 1, 2]), np.array([1, 0, 2, 1]), 3, 3),
        "path": (np.array([0, 1]), np.array([1, 2]), 3, 3),
        "empty": (np.zeros(0, np.int64), np.zeros(0, np.int64), 3, 3),
    }
    s, t = refrng.random_graph(17, 120, 21)  # test_edge_index.cpp:96-104
    cases["rand17"] = (s, t, 17, 17)
    rng = np.random.default_rng(1234)
    n = 2500
    hub_dst = np.concatenate([np.full(5200, 7), np.full(1300, 1999), rng.integers(0, n, 9000)])
    hub_src = rng.integers(0, n, hub_dst.size)
    order = rng.permutation(hub_dst.size)
    cases["hubs"] = (hub_src[order], hub_dst[order], n, n)
    for name, (src, dst, ns, nd) in cases.items():
        src = np.asarray(src, np.int64)
        dst = np.asarray(dst, np.int64)
        d[f"{name}_src"], d[f"{name}_dst"] = src, dst
        d[f"{name}_n"] = np.array([ns, nd], np.int64)
        for kind, (k, v, rows) in {"csr": (src, dst, ns), "csc": (dst, src, nd)}.items():
            rp, col, perm = ref.build_compressed(k, v, rows)
            d[f"{name}_{kind}_rowptr"], d[f"{name}_{kind}_col"], d[f"{name}_{kind}_perm"] = rp, col, perm
    return d


def spmm_fixtures(ref: Reference) -> dict:
    d = {}
    # test_message_passing.cpp:67-90
    src, dst = refrng.random_graph(12, 40, 61)
    x = refrng.random_tensor((12, 5), 62)
    w = refrng.random_tensor((40,), 63)
    d.update(ref12_src=src, ref12_dst=dst, ref12_x=x, ref12_w=w)
    for weighted in (False, True):
        for mean in (False, True):
            d[f"ref12_out_w{int(weighted)}_m{int(mean)}"] = ref.spmm(src, dst, 12, 12, x, w if weighted else None, mean)
    # test_message_passing.cpp:107-122 (undirected, asymmetric weights, exact)
    us, ud = np.array([0, 1, 1, 2, 2, 0]), np.array([1, 0, 2, 1, 0, 2])
    ux = refrng.random_tensor((3, 2), 68)
    uw = np.array([1, 10, 100, 1000, 10000, 100000], np.float64)
    d.update(und_src=us, und_dst=ud, und_x=ux, und_w=uw,
             und_out=ref.spmm(us, ud, 3, 3, ux, uw, False, undirected=True),
             und_out_unweighted=ref.spmm(us, ud, 3, 3, ux, None, False, undirected=True))
    # test_aggregate.cpp:127-134 (max routes to the first attaining position)
    vals = np.array([[5.0], [5.0], [1.0]])
    mo, ma = ref.max_path(np.array([0, 1, 2]), np.array([0, 0, 0]), 3, 1, vals)
    d.update(tie_x=vals, tie_out=mo, tie_arg=ma)
    # test_aggregate.cpp:57-66 (every kind vs naive oracle), f32 instantiation
    av = refrng.random_tensor((60, 3), 31, dtype=np.float32)
    ai = refrng.random_index(60, 7, 32)
    d.update(agg_values=av, agg_index=ai)
    for kind in ("sum", "mean", "max", "min"):
        d[f"agg_out_{kind}"] = ref.aggregate(av, ai, 7, kind)

    # synthetic f32, odd width (f=7 -> 4-byte vectors), uniform
    rng = np.random.default_rng(99)
    n, e, f = 300, 3000, 7
    s = rng.integers(0, n, e)
    t = rng.integers(0, n, e)
    x = rng.uniform(-1, 1, (n, f)).astype(np.float32)
    w = rng.uniform(0.5, 1.5, e).astype(np.float32)
    d.update(uni_src=s, uni_dst=t, uni_x=x, uni_w=w)
    for weighted in (False, True):
        for mean in (False, True):
            d[f"uni_out_w{int(weighted)}_m{int(mean)}"] = ref.spmm(s, t, n, n, x, w if weighted else None, mean)
    for kind in ("max", "min"):
        o, a = ref.max_path(s, t, n, n, x, is_min=(kind == "min"))
        d[f"uni_{kind}_out"], d[f"uni_{kind}_arg"] = o, a

    # hubs (heavy path + big-row sort), quantised features (ties, +-0), f=12
    rng = np.random.default_rng(1234)
    n = 2500
    hub_dst = np.concatenate([np.full(5200, 7), np.full(1300, 1999), rng.integers(0, n, 9000)])
    hub_src = rng.integers(0, n, hub_dst.size)
    order = rng.permutation(hub_dst.size)
    hs, ht = hub_src[order], hub_dst[order]
    f = 12
    hx = np.floor(rng.uniform(-1, 1, (n, f)) * 8) / 8
    hx[rng.random((n, f)) < 0.1] = -0.0
    hx = hx.astype(np.float32)
    d.update(hub_src=hs, hub_dst=ht, hub_x=hx)
    for mean in (False, True):
        d[f"hub_out_m{int(mean)}"] = ref.spmm(hs, ht, n, n, hx, None, mean)
    for kind in ("max", "min"):
        o, a = ref.max_path(hs, ht, n, n, hx, is_min=(kind == "min"))
        d[f"hub_{kind}_out"], d[f"hub_{kind}_arg"] = o, a
    # GCN aggregate on the hub graph with smooth features (f=16)
    gx = rng.uniform(-1, 1, (n, 16)).astype(np.float32)
    d.update(hub_gcn_x=gx, hub_gcn_out=ref.gcn_aggregate(hs, ht, n, gx))
    # bf16-rounded inputs, fp32 reference accumulate (output rounding done by the test)
    bx = bf16_round(rng.uniform(-1, 1, (n, 16)))
    d.update(hub_bf16_x=bx, hub_bf16_out=ref.spmm(hs, ht, n, n, bx, None, False))
    # spmm gradients (test_message_passing.cpp:92-105): graph salt 64, coeff 65, x 66, w 67,
    # loss = sum(spmm * coeff) -> the gradient entering spmm's closure is coeff
    bs, bd = refrng.random_graph(8, 20, 64)
    coeff = refrng.random_tensor((8, 3), 65)
    bx = refrng.random_tensor((8, 3), 66)
    bw = refrng.random_tensor((20,), 67)
    d.update(bwd_src=bs, bwd_dst=bd, bwd_g=coeff, bwd_x=bx, bwd_w=bw)
    for mean in (0, 1):
        dx, dw = ref.spmm_backward(bs, bd, 8, 8, bx, coeff, bw, bool(mean))
        d[f"bwd_dx_m{mean}"], d[f"bwd_dw_m{mean}"] = dx, dw
        dx0, _ = ref.spmm_backward(bs, bd, 8, 8, bx, coeff, None, bool(mean))
        d[f"bwd_dx_unweighted_m{mean}"] = dx0
    # larger f32 backward on the uniform graph
    ug = rng.uniform(-1, 1, (300, 7)).astype(np.float32)
    d.update(uni_g=ug)
    for mean in (0, 1):
        dx, dw = ref.spmm_backward(d["uni_src"], d["uni_dst"], 300, 300, d["uni_x"], ug, d["uni_w"], bool(mean))
        d[f"uni_bwd_dx_m{mean}"], d[f"uni_bwd_dw_m{mean}"] = dx, dw
    # GCN edge cases: test_message_passing.cpp:188-207 (edgeless -> identity norm)
    ex = refrng.random_tensor((4, 3), 74, dtype=np.float32)
    d.update(gcn_edgeless_x=ex, gcn_edgeless_out=ref.gcn_aggregate(np.zeros(0), np.zeros(0), 4, ex))
    return d


def gemm_fixtures(ref: Reference) -> dict:
    d = {}
    # test_hetero.cpp:61-73
    h0 = refrng.random_tensor((2, 3), 201)
    h1 = refrng.random_tensor((4, 3), 202)
    w = refrng.random_tensor((2, 3, 5), 203)
    x = np.concatenate([h0, h1])
    d.update(gm_x=x, gm_ptr=np.array([0, 2, 6]), gm_w=w, gm_out=ref.grouped_matmul(x, [0, 2, 6], w))
    # empty group (test_hetero.cpp:82-92)
    h = refrng.random_tensor((2, 3), 206)
    w2 = refrng.random_tensor((2, 3, 4), 207)
    d.update(gm_empty_x=h, gm_empty_w=w2, gm_empty_out=ref.grouped_matmul(h, [0, 0, 2], w2))
    # bf16-shaped case: K=N=128, ragged groups, bf16-rounded inputs, fp64 reference
    rng = np.random.default_rng(5)
    ptr = np.array([0, 300, 301, 301, 777], np.int64)
    gx = bf16_round(rng.uniform(-1, 1, (int(ptr[-1]), 128))).astype(np.float64)
    gw = bf16_round(rng.uniform(-0.1, 0.1, (4, 128, 128))).astype(np.float64)
    d.update(seg_x=gx.astype(np.float32), seg_ptr=ptr, seg_w=gw.astype(np.float32),
             seg_out64=ref.grouped_matmul(gx, ptr, gw))
    return d


def hetero_fixtures(ref: Reference) -> dict:
    """to_hetero(sage) + hetero_propagate(sum) (hetero.hpp:217-365), 3 node types,
    4 edge types (one self-relation, one node type with two incoming relations,
    one node type with none)."""
    rng = np.random.default_rng(77)
    counts = [300, 500, 20, 9]  # n3 has no incoming edge type
    node_ptr = np.concatenate([[0], np.cumsum(counts)])
    f_in, f_out = 64, 32
    h = rng.uniform(-1, 1, (node_ptr[-1], f_in)).astype(np.float32)
    ets = [(1, 0, 3000), (0, 0, 2000), (0, 2, 800), (1, 2, 500)]
    src, dst, e_ptr = [], [], [0]
    for s_t, d_t, e in ets:
        src.append(rng.integers(0, counts[s_t], e))
        dst.append(rng.integers(0, counts[d_t], e))
        e_ptr.append(e_ptr[-1] + e)
    src, dst = np.concatenate(src), np.concatenate(dst)
    w_neigh = rng.uniform(-0.125, 0.125, (len(ets), f_in, f_out)).astype(np.float32)
    w_self = rng.uniform(-0.125, 0.125, (len(counts), f_in, f_out)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, (len(counts), f_out)).astype(np.float32)
    et_src = np.array([e[0] for e in ets], np.int32)
    et_dst = np.array([e[1] for e in ets], np.int32)
    out = ref.hetero_sage(node_ptr, h, et_src, et_dst, e_ptr, src, dst, w_neigh, w_self, bias)
    return dict(node_ptr=node_ptr, h=h, et_src=et_src, et_dst=et_dst, e_ptr=np.array(e_ptr), src=src, dst=dst,
                w_neigh=w_neigh, w_self=w_self, bias=bias, out=out)


def maxbwd_fixtures(ref: Reference) -> dict:
    """Backward of the layer max/min path through the reference's own tape
    (aggregate.hpp:295-308 + gather_rows adjoint): quantised features (ties,
    +-0), a source hub (out-degree > the 1024-edge heavy threshold of the
    source view), a destination hub, duplicate edges, empty rows; f32 and f64."""
    d = {}
    rng = np.random.default_rng(4321)
    n = 3000
    src = np.concatenate([np.full(4000, 11), rng.integers(0, n, 14000), np.full(1500, 2222)])
    dst = np.concatenate([rng.integers(0, n, 4000), rng.integers(0, n - 100, 14000), rng.integers(0, 40, 1500)])
    dup = rng.integers(0, src.size, 800)
    src, dst = np.concatenate([src, src[dup]]), np.concatenate([dst, dst[dup]])
    order = rng.permutation(src.size)
    src, dst = src[order].astype(np.int64), dst[order].astype(np.int64)
    d.update(src=src, dst=dst, n=np.array([n]))
    for dt, f in (("f32", 12), ("f64", 5)):
        x = np.floor(rng.uniform(-1, 1, (n, f)) * 8) / 8
        x[rng.random((n, f)) < 0.1] = -0.0
        g = rng.uniform(-1, 1, (n, f))
        npdt = np.float32 if dt == "f32" else np.float64
        x, g = x.astype(npdt), g.astype(npdt)
        d[f"{dt}_x"], d[f"{dt}_g"] = x, g
        for kind in ("max", "min"):
            d[f"{dt}_{kind}_dx"] = ref.max_backward(src, dst, n, n, x, g, is_min=(kind == "min"))
            d[f"{dt}_{kind}_arg"] = ref.max_path(src, dst, n, n, x, is_min=(kind == "min"))[1]
    return d


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Reference()
    fixtures = (("csr", csr_fixtures), ("spmm", spmm_fixtures), ("gemm", gemm_fixtures),
                ("hetero", hetero_fixtures), ("maxbwd", maxbwd_fixtures))
    only = sys.argv[sys.argv.index("--only") + 1].split(",") if "--only" in sys.argv else None
    for name, fn in fixtures:
        if only and name not in only:
            continue
        data = fn(ref)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{path}: {len(data)} arrays, {os.path.getsize(path) / 1024:.0f} KiB")


def dataset_fixtures() -> None:
    """tests/golden/dataset_{f32,f64}: written by the reference's OWN
    save_dataset (oracle/ref_dataset_gen.cpp, `make -C oracle ref-dataset`)."""
    import shutil
    import subprocess
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref-dataset"], check=True)
    outs = [os.path.join(OUT, "dataset_f32"), os.path.join(OUT, "dataset_f64")]
    for o in outs:
        shutil.rmtree(o, ignore_errors=True)
    subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_dataset_gen"), *outs], check=True)


if __name__ == "__main__":
    if "--dataset" in sys.argv:
        dataset_fixtures()
    else:
        main()
