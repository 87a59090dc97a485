"""ctypes wrappers of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker (never as the thing
measured or shipped).

* ``Oracle``     -> oracle/liboracle.so, the plain-C restatement (gm_oracle.c);
                    travels to the GPU box.
* ``Reference``  -> oracle/_ref/libgraphmill_ref.so, the UNMODIFIED reference
                    compiled in place (oracle/Makefile); present wherever it was
                    built (it is git-ignored but shipped with the gpurun snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgraphmill_ref.so")
REF_SRC = "/root/reference/proj"

_P = C.c_void_p
_I = C.c_int64


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_oracle(with_ref: bool = True) -> None:
    """Compile the restatement (always) and the in-place reference build when
    /root/reference is present (it is absent on the GPU box)."""
    subprocess.run(["make", "-C", HERE, "liboracle"], check=True, capture_output=True)
    if with_ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Oracle:
    """The plain-C restatement (gm_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build_oracle(with_ref=False)
        self.lib = C.CDLL(ORACLE_SO)
        for name in ("or_build_compressed", "or_spmm_f32", "or_spmm_f64", "or_spmm_coo_f32",
                     "or_spmm_coo_f64", "or_spmm_max_f32", "or_spmm_max_f64", "or_gcn_norm_f32",
                     "or_gcn_norm_f64", "or_degree", "or_segment_matmul_f64", "or_segment_matmul_f32",
                     "or_spmm_backward_f32", "or_spmm_backward_f64", "or_spmm_max_backward_f32",
                     "or_spmm_max_backward_f64"):
            getattr(self.lib, name).restype = None

    def build_compressed(self, keys, values, num_rows):
        keys, values = _i64(keys), _i64(values)
        e = keys.size
        rowptr = np.zeros(num_rows + 1, np.int64)
        col = np.zeros(e, np.int64)
        perm = np.zeros(e, np.int64)
        self.lib.or_build_compressed(_ptr(keys), _ptr(values), _I(e), _I(num_rows), _ptr(rowptr),
                                     _ptr(col), _ptr(perm))
        return rowptr, col, perm

    def spmm(self, rowptr, col, perm, x, w_coo=None, mean=False, rows=None):
        """Per destination row of the grouping (rowptr/col/perm)."""
        x = np.ascontiguousarray(x)
        suf = "f64" if x.dtype == np.float64 else "f32"
        f = x.shape[1]
        n_rows = rowptr.size - 1
        rows_a = None if rows is None else _i64(rows)
        count = n_rows if rows is None else rows_a.size
        out = np.zeros((count, f), x.dtype)
        w = None if w_coo is None else np.ascontiguousarray(w_coo, dtype=x.dtype)
        getattr(self.lib, "or_spmm_" + suf)(_ptr(_i64(rowptr)), _ptr(_i64(col)), _ptr(_i64(perm)),
                                            _I(n_rows), _ptr(x), _I(f), _ptr(w), C.c_int(int(mean)),
                                            _ptr(rows_a), _I(count), _ptr(out))
        return out

    def spmm_coo(self, src, dst, n_dst, x, w, mean=False):
        x = np.ascontiguousarray(x)
        suf = "f64" if x.dtype == np.float64 else "f32"
        f = x.shape[1]
        out = np.zeros((n_dst, f), x.dtype)
        w = np.ascontiguousarray(w, dtype=x.dtype)
        getattr(self.lib, "or_spmm_coo_" + suf)(_ptr(_i64(src)), _ptr(_i64(dst)), _I(len(src)), _I(n_dst),
                                                _ptr(x), _I(f), _ptr(w), C.c_int(int(mean)), _ptr(out))
        return out

    def spmm_max_backward(self, rowptr, col, perm, arg, g, n_src):
        """dx of the max/min path from the CSC, the COO-id argmax and the output gradient."""
        g = np.ascontiguousarray(g)
        suf = "f64" if g.dtype == np.float64 else "f32"
        f = g.shape[1]
        dx = np.zeros((n_src, f), g.dtype)
        getattr(self.lib, "or_spmm_max_backward_" + suf)(_ptr(_i64(rowptr)), _ptr(_i64(col)), _ptr(_i64(perm)),
                                                         _I(rowptr.size - 1), _ptr(_i64(arg)), _ptr(g), _I(f),
                                                         _I(n_src), _ptr(dx))
        return dx

    def spmm_max(self, rowptr, col, perm, x, w_coo=None, is_min=False, rows=None):
        x = np.ascontiguousarray(x)
        suf = "f64" if x.dtype == np.float64 else "f32"
        f = x.shape[1]
        n_rows = rowptr.size - 1
        rows_a = None if rows is None else _i64(rows)
        count = n_rows if rows is None else rows_a.size
        out = np.zeros((count, f), x.dtype)
        arg = np.zeros((count, f), np.int64)
        w = None if w_coo is None else np.ascontiguousarray(w_coo, dtype=x.dtype)
        getattr(self.lib, "or_spmm_max_" + suf)(_ptr(_i64(rowptr)), _ptr(_i64(col)), _ptr(_i64(perm)),
                                                _I(n_rows), _ptr(x), _I(f), _ptr(w), C.c_int(int(is_min)),
                                                _ptr(rows_a), _I(count), _ptr(out), _ptr(arg))
        return out, arg

    def gcn_norm(self, base_src, base_dst, n_src, n_dst, g_src, g_dst, square=True, dtype=np.float32):
        suf = "f64" if dtype == np.float64 else "f32"
        g_src, g_dst = _i64(g_src), _i64(g_dst)
        norm = np.zeros(g_src.size, dtype)
        getattr(self.lib, "or_gcn_norm_" + suf)(_ptr(_i64(base_src)), _ptr(_i64(base_dst)), _I(len(base_dst)),
                                                _I(n_src), _I(n_dst), _ptr(g_src), _ptr(g_dst),
                                                _I(g_src.size), C.c_int(int(square)), _ptr(norm))
        return norm

    def spmm_backward(self, src, dst, n_src, n_dst, g, x, w_coo=None, mean=False):
        """dx, dw of spmm (message_passing.hpp:119-166) via the CSR by source."""
        src, dst = _i64(src), _i64(dst)
        g = np.ascontiguousarray(g)
        x = np.ascontiguousarray(x, dtype=g.dtype)
        suf = "f64" if g.dtype == np.float64 else "f32"
        f = g.shape[1]
        rp, col, perm = self.build_compressed(src, dst, n_src)
        deg = self.degree(dst, n_dst) if mean else None
        dx = np.zeros((n_src, f), g.dtype)
        w = None if w_coo is None else np.ascontiguousarray(w_coo, dtype=g.dtype)
        dw = np.zeros(src.size, g.dtype) if w is not None else None
        getattr(self.lib, "or_spmm_backward_" + suf)(
            _ptr(rp), _ptr(col), _ptr(perm), _I(n_src), _ptr(src), _ptr(dst), _I(src.size), _ptr(g), _ptr(x),
            _I(f), _ptr(w), _ptr(deg), _ptr(dx), _ptr(dw))
        return dx, dw

    def degree(self, ids, n):
        deg = np.zeros(n, np.int64)
        ids = _i64(ids)
        self.lib.or_degree(_ptr(ids), _I(ids.size), _I(n), _ptr(deg))
        return deg

    def segment_matmul(self, x, ptr, w):
        x = np.ascontiguousarray(x)
        w = np.ascontiguousarray(w, dtype=x.dtype)
        suf = "f64" if x.dtype == np.float64 else "f32"
        g, k, n = w.shape
        out = np.zeros((x.shape[0], n), x.dtype)
        getattr(self.lib, "or_segment_matmul_" + suf)(_ptr(x), _ptr(_i64(ptr)), _I(g), _I(k), _I(n),
                                                      _ptr(w), _ptr(out))
        return out

    # composite: the GCN fused branch (message_passing.hpp:490-495) restated
    def gcn_aggregate(self, src, dst, n, xw):
        src, dst = _i64(src), _i64(dst)
        loops = np.arange(n, dtype=np.int64)
        g_src = np.concatenate([src, loops])
        g_dst = np.concatenate([dst, loops])
        norm = self.gcn_norm(src, dst, n, n, g_src, g_dst, True, xw.dtype)
        rowptr, col, perm = self.build_compressed(g_dst, g_src, n)
        return self.spmm(rowptr, col, perm, xw, w_coo=norm)


class Reference:
    """The reference itself (oracle/_ref/libgraphmill_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} not built (needs /root/reference; see oracle/Makefile)")
        self.lib = C.CDLL(REF_SO)
        self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, st):
        if st == 0:
            return
        msg = self.lib.ref_last_error().decode()
        if st == 2:
            raise IndexError(msg)
        if st == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    def build_compressed(self, keys, values, num_rows):
        keys, values = _i64(keys), _i64(values)
        e = keys.size
        rowptr = np.zeros(num_rows + 1, np.int64)
        col = np.zeros(e, np.int64)
        perm = np.zeros(e, np.int64)
        self._check(self.lib.ref_build_compressed(_ptr(keys), _ptr(values), _I(e), _I(num_rows),
                                                  _ptr(rowptr), _ptr(col), _ptr(perm)))
        return rowptr, col, perm

    def edge_index_check(self, src, dst, n_src, n_dst, undirected=False, sort_order=0):
        src, dst = _i64(src), _i64(dst)
        self._check(self.lib.ref_edge_index_check(_ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst),
                                                  C.c_int(int(undirected)), C.c_int(sort_order)))

    def spmm(self, src, dst, n_src, n_dst, x, w=None, mean=False, undirected=False):
        x = np.ascontiguousarray(x)
        suf = "f64" if x.dtype == np.float64 else "f32"
        src, dst = _i64(src), _i64(dst)
        f = x.shape[1]
        out = np.zeros((n_dst, f), x.dtype)
        wa = None if w is None else np.ascontiguousarray(w, dtype=x.dtype)
        self._check(getattr(self.lib, "ref_spmm_" + suf)(
            _ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst), C.c_int(int(undirected)), _ptr(x), _I(f),
            _ptr(wa), C.c_int(int(mean)), _ptr(out)))
        return out

    def spmm_backward(self, src, dst, n_src, n_dst, x, g, w=None, mean=False, undirected=False):
        x = np.ascontiguousarray(x)
        g = np.ascontiguousarray(g, dtype=x.dtype)
        suf = "f64" if x.dtype == np.float64 else "f32"
        src, dst = _i64(src), _i64(dst)
        f = x.shape[1]
        dx = np.zeros((n_src, f), x.dtype)
        wa = None if w is None else np.ascontiguousarray(w, dtype=x.dtype)
        dw = None if w is None else np.zeros(src.size, x.dtype)
        self._check(getattr(self.lib, "ref_spmm_backward_" + suf)(
            _ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst), C.c_int(int(undirected)), _ptr(x), _I(f),
            _ptr(wa), C.c_int(int(mean)), _ptr(g), _ptr(dx), _ptr(dw)))
        return dx, dw

    def max_path(self, src, dst, n_src, n_dst, x, is_min=False):
        x = np.ascontiguousarray(x)
        suf = "f64" if x.dtype == np.float64 else "f32"
        src, dst = _i64(src), _i64(dst)
        f = x.shape[1]
        out = np.zeros((n_dst, f), x.dtype)
        arg = np.zeros((n_dst, f), np.int64)
        self._check(getattr(self.lib, "ref_max_" + suf)(
            _ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst), _ptr(x), _I(f), C.c_int(int(is_min)),
            _ptr(out), _ptr(arg)))
        return out, arg

    def max_backward(self, src, dst, n_src, n_dst, x, g, is_min=False):
        """dx of the layer max/min path through the reference's own tape."""
        x = np.ascontiguousarray(x)
        g = np.ascontiguousarray(g, dtype=x.dtype)
        suf = "f64" if x.dtype == np.float64 else "f32"
        src, dst = _i64(src), _i64(dst)
        f = x.shape[1]
        dx = np.zeros((n_src, f), x.dtype)
        self._check(getattr(self.lib, "ref_max_backward_" + suf)(
            _ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst), _ptr(x), _I(f), C.c_int(int(is_min)),
            _ptr(g), _ptr(dx)))
        return dx

    def aggregate(self, values, index, n, kind):
        values = np.ascontiguousarray(values, dtype=np.float32)
        if values.ndim == 1:
            values = values.reshape(-1, 1)
        index = _i64(index)
        out = np.zeros((n, values.shape[1]), np.float32)
        k = {"sum": 0, "mean": 1, "max": 2, "min": 3}[kind]
        self._check(self.lib.ref_aggregate_f32(_ptr(values), _I(values.shape[0]), _I(values.shape[1]),
                                               _ptr(index), _I(n), C.c_int(k), _ptr(out)))
        return out

    def gcn_aggregate(self, src, dst, n, xw):
        xw = np.ascontiguousarray(xw, dtype=np.float32)
        src, dst = _i64(src), _i64(dst)
        out = np.zeros_like(xw)
        self._check(self.lib.ref_gcn_aggregate_f32(_ptr(src), _ptr(dst), _I(src.size), _I(n), _ptr(xw),
                                                   _I(xw.shape[1]), _ptr(out)))
        return out

    def gcn_layer(self, src, dst, n, h, w, b):
        h = np.ascontiguousarray(h, dtype=np.float32)
        w = np.ascontiguousarray(w, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        src, dst = _i64(src), _i64(dst)
        out = np.zeros((n, w.shape[1]), np.float32)
        self._check(self.lib.ref_gcn_layer_f32(_ptr(src), _ptr(dst), _I(src.size), _I(n), _ptr(h),
                                               _I(h.shape[1]), _ptr(w), _ptr(b), _I(w.shape[1]), _ptr(out)))
        return out

    def gcn_model(self, src, dst, n, h, layers, dtype=np.float32):
        """Model<S>::forward of a GCN stack (message_passing.hpp:631-641):
        layers = [(W [f_in, f_out], b [f_out]), ...], relu between layers."""
        h = np.ascontiguousarray(h, dtype=dtype)
        dims = np.array([h.shape[1]] + [w.shape[1] for w, _ in layers], np.int64)
        ws = np.ascontiguousarray(np.concatenate([np.asarray(w, dtype).ravel() for w, _ in layers]))
        bs = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype).ravel() for _, b in layers]))
        src, dst = _i64(src), _i64(dst)
        out = np.zeros((n, dims[-1]), dtype)
        suf = "f64" if dtype == np.float64 else "f32"
        self._check(getattr(self.lib, "ref_gcn_model_" + suf)(
            _ptr(src), _ptr(dst), _I(src.size), _I(n), _ptr(h), C.c_int32(len(layers)), _ptr(dims), _ptr(ws),
            _ptr(bs), _ptr(out)))
        return out

    def grouped_matmul(self, x, ptr, w):
        x = np.ascontiguousarray(x)
        w = np.ascontiguousarray(w, dtype=x.dtype)
        suf = "f64" if x.dtype == np.float64 else "f32"
        g, k, n = w.shape
        out = np.zeros((x.shape[0], n), x.dtype)
        self._check(getattr(self.lib, "ref_grouped_matmul_" + suf)(
            _ptr(x), _ptr(_i64(ptr)), _I(g), _I(k), _I(n), _ptr(w), _ptr(out)))
        return out

    def hetero_sage(self, node_ptr, h, et_src, et_dst, e_ptr, src, dst, w_neigh, w_self, bias):
        """to_hetero(sage) + hetero_propagate(sum), node types n<i>, edge types (n<s>, r<i>, n<d>)."""
        h = np.ascontiguousarray(h, dtype=np.float32)
        f_in = h.shape[1]
        f_out = w_self.shape[2]
        out = np.zeros((h.shape[0], f_out), np.float32)
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
        f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
        es, ed = i32(et_src), i32(et_dst)
        self._check(self.lib.ref_hetero_sage_f32(
            C.c_int32(len(node_ptr) - 1), _ptr(_i64(node_ptr)), _ptr(h), _I(f_in), _I(f_out), C.c_int32(len(es)),
            _ptr(es), _ptr(ed), _ptr(_i64(e_ptr)), _ptr(_i64(src)), _ptr(_i64(dst)), _ptr(f32(w_neigh)),
            _ptr(f32(w_self)), _ptr(f32(bias)), _ptr(out)))
        return out

    def bench_spmm(self, src, dst, n_src, n_dst, x, mean=False, threads=1, rows_limit=0, warmup=1,
                   repeat=3):
        """Reference spmm<float> timed by its own time_loop over `threads` row ranges."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        src, dst = _i64(src), _i64(dst)
        secs = C.c_double(0)
        edges = C.c_int64(0)
        self._check(self.lib.ref_bench_spmm_f32(
            _ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst), _ptr(x), _I(x.shape[1]),
            C.c_int(int(mean)), C.c_int(threads), _I(rows_limit), C.c_int(warmup), C.c_int(repeat),
            C.byref(secs), C.byref(edges)))
        return secs.value, edges.value

    # -- synthetic inputs without the product library -------------
    def synth_edges(self, kind, seed, count, n_src, n_dst, first=0, threads=None):
        src = np.zeros(count, np.int64)
        dst = np.zeros(count, np.int64)
        self._check(self.lib.ref_synth_edges(C.c_int(kind), C.c_uint64(seed), _I(first), _I(count), _I(n_src),
                                             _I(n_dst), _ptr(src), _ptr(dst), C.c_int(threads or host_threads())))
        return src, dst

    def synth_features(self, seed, rows, f, quantize=0, first_row=0, threads=None):
        x = np.zeros((rows, f), np.float32)
        self._check(self.lib.ref_synth_features_f32(C.c_uint64(seed), _I(first_row), _I(rows), _I(f),
                                                    C.c_int(quantize), _ptr(x), C.c_int(threads or host_threads())))
        return x

    def bench_build_compressed(self, keys, values, num_rows):
        """Seconds of one reference build_compressed (edge_index.cpp:45-62), 1 thread."""
        secs = C.c_double(0)
        keys, values = _i64(keys), _i64(values)
        self._check(self.lib.ref_bench_build_compressed(_ptr(keys), _ptr(values), _I(keys.size), _I(num_rows),
                                                        C.byref(secs)))
        return secs.value

    def bench_max(self, src, dst, n_src, n_dst, x, rows_limit=0):
        """Seconds of one reference max path (message_passing.hpp:508-514) over the
        first rows_limit destination rows, 1 thread; returns (seconds, edges)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        src, dst = _i64(src), _i64(dst)
        secs = C.c_double(0)
        edges = C.c_int64(0)
        self._check(self.lib.ref_bench_max_f32(_ptr(src), _ptr(dst), _I(src.size), _I(n_src), _I(n_dst), _ptr(x),
                                               _I(x.shape[1]), _I(rows_limit), C.byref(secs), C.byref(edges)))
        return secs.value, edges.value


def host_threads() -> int:
    """Host cores this process may run on (the CPU arms' thread count)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"

