"""Host-side mirror of the reference operator API over the C-ABI.

Names, argument meaning and error behaviour follow the reference graphmill
engine (/root/reference/proj/include/graphmill/*.hpp) so a test written
against the reference reads the same here:

    EdgeIndex(src, dst, num_src_nodes, num_dst_nodes, sort_order=, is_undirected=)
        .to_csr() / .to_csc() / .transpose_view()   edge_index.hpp:43-116
    build_compressed(keys, values, num_rows)          edge_index.hpp:120-121
    spmm(e, x, edge_weight, reduce)                   message_passing.hpp:92-169
    neighbor_aggregate(e, x, kind, ...)               message_passing.hpp:500-514 (sum/mean/max/min)
    spmm_backward(e, x, w, reduce, grad_out)          message_passing.hpp:119-166 (dx, dw)
    gcn_aggregate(e, xw) / gcn_layer(e, h, W, b)      message_passing.hpp:437-463, 490-499
    aggregate(values, index, num_groups, kind)        aggregate.hpp:154-215
    segment_matmul(x, ptr, W) / grouped_matmul(xs, W) hetero.hpp:134-157

Device memory, streams and the collective plumbing come from PyTorch; every
computation on the path runs in libgraphmill_b200.so. std::invalid_argument
maps to ValueError, std::out_of_range to IndexError.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _lib as L

_DT = {torch.float32: L.GM_F32, torch.float64: L.GM_F64, torch.bfloat16: L.GM_BF16}
_KIND = {"sum": L.GM_SUM, "mean": L.GM_MEAN, "max": L.GM_MAX, "min": L.GM_MIN}


def _p(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _same_device(where: str, device, *tensors) -> None:
    """Every kernel argument must live in the device memory of the index (or
    of the first operand): a host tensor here would reach the kernels as a host
    pointer. The reference has no devices; this is the mirror's own check."""
    if device is None or device.type != "cuda":
        raise ValueError(f"{where}: CUDA tensors required (got {device})")
    for t in tensors:
        if t is not None and t.device != device:
            raise ValueError(f"{where}: all tensors must be on {device} (got {t.device})")


def _dev_index(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int64).contiguous()
    return torch.as_tensor(list(a), dtype=torch.int64, device=device)


@dataclass
class CsrView:
    """Device CSR (edge_index.hpp:22-29): rowptr int64[n+1], col/perm int32[nnz]."""

    rowptr: torch.Tensor
    col: torch.Tensor
    perm: torch.Tensor
    num_cols: int
    nnz: Optional[int] = None  # edges of these rows (set for row slices of a larger CSR)
    _plan: Optional[dict] = field(default=None, repr=False)

    def num_rows(self) -> int:
        return self.rowptr.numel() - 1

    def num_entries(self) -> int:
        return self.col.numel() if self.nnz is None else self.nnz

    def row_slice(self, r0: int, r1: int, nnz: int) -> "CsrView":
        """Rows [r0, r1) sharing col/perm (offsets stay global); nnz = their edge count."""
        return CsrView(self.rowptr[r0:r1 + 1], self.col, self.perm, self.num_cols, nnz)

    def c_struct(self) -> L.gm_csr:
        return L.gm_csr(self.num_rows(), self.num_cols, self.num_entries(),
                        self.rowptr.data_ptr(), self.col.data_ptr(), self.perm.data_ptr())

    def plan(self, row_bytes: int = 0):
        """Scheduling metadata (gm_spmm_plan), built once per row-width class
        and cached: rows >= 1 KB wide (F=602 fp32) raise the hub threshold to
        4096 in-edges and keep 256-entry windows; narrower rows keep the
        default 1024 threshold and the library's automatic window size."""
        thr = 4096 if row_bytes >= 1024 else 0
        if self._plan is None:
            self._plan = {}
        if thr not in self._plan:
            lib = L.lib()
            nbytes = lib.gm_spmm_plan_bytes(self.num_rows(), self.num_cols, self.num_entries())
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.rowptr.device)
            plan = L.gm_spmm_plan()
            plan.heavy_threshold = thr
            plan.window_edges = 256 if row_bytes >= 1024 else 0  # wide rows: short windows (0 = auto)
            csr = self.c_struct()
            L.check(lib.gm_spmm_plan_build(C.byref(csr), _p(buf), nbytes, C.byref(plan), _stream()),
                    "gm_spmm_plan_build")
            self._plan[thr] = (plan, buf)
        return self._plan[thr][0]

    def entry_rows(self) -> torch.Tensor:
        """Per-entry row id (int32, from the view's first entry), cached beside the view."""
        er = getattr(self, "_entry_rows", None)
        if er is None:
            er = torch.empty(max(self.num_entries(), 1), dtype=torch.int32, device=self.rowptr.device)
            cs = self.c_struct()
            L.check(L.lib().gm_csr_entry_rows(C.byref(cs), _p(er), _stream()), "gm_csr_entry_rows")
            self._entry_rows = er
        return er

    def to_host(self):
        """(rowptr, col, perm) as int64 CPU tensors, the reference's CsrView layout."""
        return self.rowptr.cpu(), self.col.cpu().long(), self.perm.cpu().long()


def build_compressed(keys: torch.Tensor, values: torch.Tensor, num_rows: int,
                     num_cols: int = 0) -> CsrView:
    """edge_index.cpp:45-62 on the device (bit-exact stable counting sort)."""
    lib = L.lib()
    dev = keys.device
    e = keys.numel()
    rowptr = torch.empty(num_rows + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(e, 0), dtype=torch.int32, device=dev)
    perm = torch.empty(max(e, 0), dtype=torch.int32, device=dev)
    ws_bytes = lib.gm_build_compressed_workspace(e, num_rows)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    L.check(lib.gm_build_compressed(_p(keys), _p(values), e, num_rows, _p(rowptr), _p(col), _p(perm),
                                    _p(ws), ws_bytes, _stream()), "gm_build_compressed")
    return CsrView(rowptr, col, perm, num_cols)


class EdgeIndex:
    """COO edge list with verified claims and demand-filled device CSR/CSC
    caches (edge_index.hpp:43-116). Copies share arrays and caches."""

    def __init__(self, src, dst, num_src_nodes: int, num_dst_nodes: int,
                 sort_order: Optional[str] = None, is_undirected: Optional[bool] = None,
                 device: str | torch.device = "cuda"):
        src_t = _dev_index(src, device)
        dst_t = _dev_index(dst, device)
        if src_t.numel() != dst_t.numel():
            raise ValueError("EdgeIndex: src and dst lengths differ")
        if num_src_nodes < 0 or num_dst_nodes < 0:
            raise ValueError("EdgeIndex: negative node count")
        self._src, self._dst = src_t, dst_t
        self._num_edges = src_t.numel()
        self._num_src, self._num_dst = int(num_src_nodes), int(num_dst_nodes)
        self._cache = _CacheSlot()
        self._verify_claims(sort_order, is_undirected)

    # -- claims (edge_index.cpp:84-119) --------------------------------------
    def _verify_claims(self, sort_order, is_undirected):
        lib = L.lib()
        ws = torch.empty(64, dtype=torch.uint8, device=self._src.device)
        L.check(lib.gm_check_index_bounds(_p(self._src), self._num_edges, self._num_src,
                                          b"EdgeIndex: src", _p(ws), _stream()), "bounds")
        L.check(lib.gm_check_index_bounds(_p(self._dst), self._num_edges, self._num_dst,
                                          b"EdgeIndex: dst", _p(ws), _stream()), "bounds")
        self._sort_order = "unsorted"
        self._undirected = False
        if sort_order not in (None, "unsorted"):
            if sort_order not in ("by_src", "by_dst"):
                raise ValueError(f"EdgeIndex: unknown sort order {sort_order}")
            keys = self._src if sort_order == "by_src" else self._dst
            pos = C.c_int64(-1)
            L.check(lib.gm_first_unsorted(_p(keys), self._num_edges, C.byref(pos), _p(ws), _stream()),
                    "first_unsorted")
            if pos.value >= 0:
                raise ValueError(f"EdgeIndex: claim {sort_order} violated at position {pos.value}")
            self._sort_order = sort_order
        if is_undirected:
            if self._num_src != self._num_dst:
                raise ValueError(
                    "EdgeIndex: is_undirected claim requires num_src_nodes == num_dst_nodes")
            bad = _first_asymmetric(self._src, self._dst, self._num_src)
            if bad >= 0:
                s, d = int(self._src[bad]), int(self._dst[bad])
                raise ValueError(f"EdgeIndex: is_undirected claim violated at position {bad} "
                                 f"(edge {s}->{d} lacks a matching reverse)")
            self._undirected = True

    # -- accessors ---------------------------------------------------------------
    def src(self) -> torch.Tensor:
        return self._src[: self._num_edges]

    def dst(self) -> torch.Tensor:
        return self._dst[: self._num_edges]

    def full_src(self) -> torch.Tensor:
        return self._src

    def full_dst(self) -> torch.Tensor:
        return self._dst

    def num_edges(self) -> int:
        return self._num_edges

    def num_src_nodes(self) -> int:
        return self._num_src

    def num_dst_nodes(self) -> int:
        return self._num_dst

    def sort_order(self) -> str:
        return self._sort_order

    def is_undirected(self) -> bool:
        return self._undirected

    def is_prefix_view(self) -> bool:
        return self._num_edges != self._src.numel()

    # -- caches (edge_index.cpp:121-145) -----------------------------------------
    def _fill_cache(self, by_dst: bool) -> CsrView:
        slot = self._cache
        hit = slot.csc if by_dst else slot.csr
        if hit is not None:
            return hit
        keys, vals, n_rows, n_cols = ((self.dst(), self.src(), self._num_dst, self._num_src) if by_dst
                                      else (self.src(), self.dst(), self._num_src, self._num_dst))
        built = build_compressed(keys, vals, n_rows, n_cols)
        with slot.lock:  # compute-then-publish: at most one result wins
            if by_dst:
                slot.csc_builds += 1
                if slot.csc is None:
                    slot.csc = built
                return slot.csc
            slot.csr_builds += 1
            if slot.csr is None:
                slot.csr = built
            return slot.csr

    def to_csr(self) -> CsrView:
        return self._fill_cache(False)

    def to_csc(self) -> CsrView:
        return self._fill_cache(True)

    def transpose_view(self) -> CsrView:
        return self.to_csr() if self._undirected else self.to_csc()

    def _exact_dst_grouping(self) -> CsrView:
        """Destination grouping for the reference's undirected+weights COO sweep
        (message_passing.hpp:51-59): cached privately, never published as the
        CSC cache (the reference never builds one there, test_message_passing.cpp:121)."""
        if self._cache.exact is None:
            self._cache.exact = build_compressed(self.dst(), self.src(), self._num_dst, self._num_src)
        return self._cache.exact

    def source_view(self) -> CsrView:
        """Per source node, its entries in ascending CSC position (gm_source_view),
        with COO edge ids as perm: the gather order of the max/min backward.
        Built once from the CSC and cached beside it."""
        if self._cache.source is None:
            # undirected indices group exactly without publishing a CSC (as the forward)
            csc = self._exact_dst_grouping() if self._undirected else self.to_csc()
            lib = L.lib()
            e, n = csc.num_entries(), self._num_src
            dev = csc.rowptr.device
            rowptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
            col = torch.empty(max(e, 1), dtype=torch.int32, device=dev)
            eid = torch.empty(max(e, 1), dtype=torch.int32, device=dev)
            nb = lib.gm_source_view_workspace(e, n)
            ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
            cs = csc.c_struct()
            L.check(lib.gm_source_view(C.byref(cs), n, _p(rowptr), _p(col), _p(eid), _p(ws), nb, _stream()),
                    "gm_source_view")
            self._cache.source = CsrView(rowptr, col, eid, self._num_dst)
        return self._cache.source

    def has_csr_cache(self) -> bool:
        return self._cache.csr is not None

    def has_csc_cache(self) -> bool:
        return self._cache.csc is not None

    def csr_build_count(self) -> int:
        return self._cache.csr_builds

    def csc_build_count(self) -> int:
        return self._cache.csc_builds

    def sort_by(self, order: str):
        """(sorted EdgeIndex, perm) — edge_index.cpp:147-188. The grouped view is
        a stable device counting sort; the new COO arrays are src[perm] /
        dst[perm]; the sorted index carries the grouping as its CSR (by_src) or
        CSC (by_dst) cache with identity perm, as the reference publishes it."""
        if order not in ("by_src", "by_dst"):
            raise ValueError("EdgeIndex: sort_by needs by_src or by_dst")
        by_src = order == "by_src"
        keys, vals = (self.src(), self.dst()) if by_src else (self.dst(), self.src())
        n_rows, n_cols = (self._num_src, self._num_dst) if by_src else (self._num_dst, self._num_src)
        grouped = build_compressed(keys, vals, n_rows, n_cols)
        e = self._num_edges
        lib = L.lib()
        new_src = torch.empty(e, dtype=torch.int64, device=self._src.device)
        new_dst = torch.empty(e, dtype=torch.int64, device=self._src.device)
        if e:
            L.check(lib.gm_permute_edge_values(L.GM_F64, _p(self.src()), _p(grouped.perm), e, _p(new_src), _stream()),
                    "permute src")
            L.check(lib.gm_permute_edge_values(L.GM_F64, _p(self.dst()), _p(grouped.perm), e, _p(new_dst), _stream()),
                    "permute dst")
        out = EdgeIndex.__new__(EdgeIndex)
        out._src, out._dst = new_src, new_dst
        out._num_edges = e
        out._num_src, out._num_dst = self._num_src, self._num_dst
        out._sort_order = order
        out._undirected = self._undirected
        out._cache = _CacheSlot()
        carried = CsrView(grouped.rowptr, grouped.col,
                          torch.arange(e, dtype=torch.int32, device=self._src.device), n_cols)
        if by_src:
            out._cache.csr = carried
        else:
            out._cache.csc = carried
        return out, grouped.perm.to(torch.int64)

    def prefix_edges(self, count: int, num_src_nodes: int, num_dst_nodes: int) -> "EdgeIndex":
        """Zero-copy view of the first `count` edges (edge_index.cpp:201-216)."""
        if count < 0 or count > self._num_edges:
            raise IndexError("EdgeIndex: prefix count out of range")
        view = EdgeIndex.__new__(EdgeIndex)
        view._src, view._dst = self._src, self._dst
        view._num_edges = count
        view._num_src, view._num_dst = num_src_nodes, num_dst_nodes
        view._sort_order = self._sort_order
        view._undirected = False
        view._cache = _CacheSlot()
        lib = L.lib()
        ws = torch.empty(64, dtype=torch.uint8, device=self._src.device)
        L.check(lib.gm_check_index_bounds(_p(view.src()), count, num_src_nodes, b"EdgeIndex: src",
                                          _p(ws), _stream()), "bounds")
        L.check(lib.gm_check_index_bounds(_p(view.dst()), count, num_dst_nodes, b"EdgeIndex: dst",
                                          _p(ws), _stream()), "bounds")
        return view


class _CacheSlot:
    def __init__(self):
        self.lock = threading.Lock()
        self.csr: Optional[CsrView] = None
        self.csc: Optional[CsrView] = None
        self.csr_builds = 0
        self.csc_builds = 0
        self.exact: Optional[CsrView] = None
        self.source: Optional[CsrView] = None
        self.gcn_deg: dict = {}


def _first_asymmetric(src: torch.Tensor, dst: torch.Tensor, n: int) -> int:
    """First COO position whose (u,v) multiplicity differs from (v,u)'s
    (edge_index.cpp:98-118): gm_first_asymmetric (device radix sort of the
    pair keys + per-position multiplicity lookups)."""
    if src.numel() == 0:
        return -1
    lib = L.lib()
    nb = lib.gm_first_asymmetric_workspace(src.numel())
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=src.device)
    pos = C.c_int64(-1)
    L.check(lib.gm_first_asymmetric(_p(src), _p(dst), src.numel(), n, C.byref(pos), _p(ws), nb, _stream()),
            "gm_first_asymmetric")
    return pos.value


# ---------------------------------------------------------------------------
# Aggregation
# ---------------------------------------------------------------------------

def _run_spmm(grouping: CsrView, x: torch.Tensor, kind: str, w_csr: Optional[torch.Tensor] = None,
              gcn: Optional[L.gm_gcn_norm] = None, want_arg: bool = False, num_rows: Optional[int] = None,
              out: Optional[torch.Tensor] = None):
    if x.dtype not in _DT:
        raise ValueError(f"spmm: unsupported dtype {x.dtype}")
    _same_device("spmm", grouping.rowptr.device, x, out, w_csr)
    x = x.contiguous()
    f = x.shape[1] if x.dim() == 2 else 1
    rows = grouping.num_rows() if num_rows is None else num_rows
    shape = (rows, f) if x.dim() == 2 else (rows,)
    if out is None:
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
    elif (tuple(out.shape) != shape or not out.is_contiguous() or out.dtype != x.dtype
          or out.device != x.device):
        raise ValueError("spmm: out must be a contiguous [num_dst_nodes, F] tensor of x's dtype and device")
    arg = torch.empty((rows, f), dtype=torch.int32, device=x.device) if want_arg else None
    csr = grouping.c_struct()
    plan = grouping.plan(row_bytes=f * x.element_size())
    L.check(L.lib().gm_spmm(C.byref(csr), C.byref(plan), _DT[x.dtype], _p(x), f, _p(w_csr),
                            C.byref(gcn) if gcn is not None else None, _KIND[kind], _p(out), _p(arg),
                            _stream()), "gm_spmm")
    return (out, arg) if want_arg else out


def _permute(values: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(values)
    L.check(L.lib().gm_permute_edge_values(_DT[values.dtype], _p(values), _p(perm), values.numel(),
                                           _p(out), _stream()), "permute")
    return out


def spmm(e: EdgeIndex, x: torch.Tensor, edge_weight: Optional[torch.Tensor], reduce: str,
         out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """message_passing.hpp:92-169 forward: out[v] = sum_{(w,v)} weight * x[w] (or mean).
    `out` (optional): a contiguous [num_dst_nodes, F] destination, e.g. a slice of
    a concatenated buffer, so callers avoid a copy."""
    if reduce not in ("sum", "mean"):
        raise ValueError("spmm: reduce must be sum or mean")
    if x.shape[0] != e.num_src_nodes():
        raise ValueError("spmm: feature rows != num_src_nodes")
    if edge_weight is not None and edge_weight.numel() != e.num_edges():
        raise ValueError("spmm: edge weight length != num_edges")
    _same_device("spmm", e.src().device, x, edge_weight)
    w_csr = None
    if edge_weight is not None:
        # Undirected + weights: the reference sweeps COO (message_passing.hpp:51-59),
        # i.e. ascending COO position per destination = CSC order.
        grouping = e._exact_dst_grouping() if e.is_undirected() else e.transpose_view()
        w_csr = _permute(edge_weight.to(_acc_dtype(x.dtype)).contiguous(), grouping.perm)
    else:
        grouping = e.transpose_view()
    return _run_spmm(grouping, x, reduce, w_csr=w_csr, num_rows=e.num_dst_nodes(), out=out)


def spmm_backward(e: EdgeIndex, x: torch.Tensor, edge_weight: Optional[torch.Tensor], reduce: str,
                  grad_out: torch.Tensor):
    """Backward of spmm (message_passing.hpp:119-166): (dx, dw). dx is the
    transposed product over the CSR-by-source cache (:143), dw the per-edge
    dot product (:156-165); mean divides the gradient by max(deg, 1) (:128-132).
    dw is None without an edge weight. f32/f64, bit-identical to the reference."""
    if reduce not in ("sum", "mean"):
        raise ValueError("spmm: reduce must be sum or mean")
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError("spmm_backward: f32/f64 only")
    if x.dim() != 2 or x.shape[0] != e.num_src_nodes():
        raise ValueError("spmm: feature rows != num_src_nodes")
    if grad_out.dim() != 2 or tuple(grad_out.shape) != (e.num_dst_nodes(), x.shape[1]):
        raise ValueError("spmm_backward: grad_out must be [num_dst_nodes, F]")
    if edge_weight is not None and edge_weight.numel() != e.num_edges():
        raise ValueError("spmm: edge weight length != num_edges")
    _same_device("spmm_backward", e.src().device, x, grad_out, edge_weight)
    lib = L.lib()
    g = grad_out.to(x.dtype).contiguous()
    f = g.shape[1]
    if reduce == "mean":
        deg = torch.empty(e.num_dst_nodes(), dtype=torch.int32, device=g.device)
        L.check(lib.gm_degree(_p(e.dst()), e.num_edges(), e.num_dst_nodes(), _p(deg), _stream()), "degree")
        gs = torch.empty_like(g)
        L.check(lib.gm_scale_rows_div(_DT[x.dtype], _p(g), g.shape[0], f, _p(deg), _p(gs), _stream()), "scale")
    else:
        gs = g
    csr = e.to_csr()
    w_csr = None
    if edge_weight is not None:
        w_csr = _permute(edge_weight.to(x.dtype).contiguous(), csr.perm)
    dx = _run_spmm(csr, gs, "sum", w_csr=w_csr, num_rows=e.num_src_nodes())
    dw = None
    if edge_weight is not None:
        # destination-grouped order (the CSC cache): each gradient row is read
        # once per row run; results land at their COO positions
        dw = torch.empty(e.num_edges(), dtype=x.dtype, device=x.device)
        csc = e.to_csc()
        cs = csc.c_struct()
        plan = csc.plan(row_bytes=f * x.element_size())
        L.check(lib.gm_edge_dot_csc(_DT[x.dtype], C.byref(cs), C.byref(plan), _p(csc.entry_rows()), _p(gs),
                                    _p(x.contiguous()), f, _p(dw), _stream()), "edge_dot_csc")
    return dx, dw


def _acc_dtype(dt):
    return torch.float64 if dt == torch.float64 else torch.float32


def neighbor_aggregate(e: EdgeIndex, x: torch.Tensor, kind: str,
                       edge_weight: Optional[torch.Tensor] = None, return_argmax: bool = False):
    """The fused segment path of layer_neighbor_aggregate (message_passing.hpp:500-514)
    for identity messages: sum/mean through spmm, max/min through
    dst_grouped_order + gather_rows + aggregate without the E x F temporary.
    return_argmax: also the COO edge id of the first attaining edge (-1 if empty)."""
    if kind not in _KIND:
        raise ValueError(f"unknown aggregation kind: {kind}")
    if x.shape[0] != e.num_src_nodes():
        raise ValueError("propagate: h_src rows != num_src_nodes")
    _same_device("neighbor_aggregate", e.src().device, x, edge_weight)
    # Undirected indices: sum/mean follow the reference's CSR order
    # (A = A^T, message_passing.hpp:47-85). max/min use the exact destination
    # grouping: the reference's dst_grouped_order would gather e.src()[perm]
    # over the CSR — the row node itself, not its neighbour (:205-212) — a
    # divergence kept deliberately so the fused path equals the edge path and
    # argmax names the forward edge (u -> v).
    maxmin = kind in ("max", "min")
    grouping = e._exact_dst_grouping() if (e.is_undirected() and maxmin) else e.transpose_view()
    w_csr = None
    if edge_weight is not None:
        w_csr = _permute(edge_weight.to(_acc_dtype(x.dtype)).contiguous(), grouping.perm)
    want = return_argmax and kind in ("max", "min")
    return _run_spmm(grouping, x, kind, w_csr=w_csr, want_arg=want, num_rows=e.num_dst_nodes())


def neighbor_aggregate_backward(e: EdgeIndex, kind: str, grad_out: torch.Tensor,
                                argmax: torch.Tensor) -> torch.Tensor:
    """Backward of neighbor_aggregate max/min (message_passing.hpp:508-514):
    aggregate's argpos scatter (aggregate.hpp:295-308) then the gather_rows
    adjoint (tensor.hpp:510-524), fused into one gather over the source view.
    argmax: the COO edge ids returned by neighbor_aggregate(..., return_argmax=True).
    Returns dx [num_src_nodes, F], bit-identical to the reference tape."""
    if kind not in ("max", "min"):
        raise ValueError("neighbor_aggregate_backward: max or min")
    if grad_out.dtype not in (torch.float32, torch.float64):
        raise ValueError("neighbor_aggregate_backward: f32/f64 only")
    if grad_out.dim() != 2 or grad_out.shape[0] != e.num_dst_nodes():
        raise ValueError("neighbor_aggregate_backward: grad_out must be [num_dst_nodes, F]")
    if tuple(argmax.shape) != tuple(grad_out.shape) or argmax.dtype != torch.int32:
        raise ValueError("neighbor_aggregate_backward: argmax must be int32 like grad_out")
    _same_device("neighbor_aggregate_backward", e.src().device, grad_out, argmax)
    g = grad_out.contiguous()
    f = g.shape[1]
    view = e.source_view()
    dx = torch.empty((e.num_src_nodes(), f), dtype=g.dtype, device=g.device)
    cs = view.c_struct()
    plan = view.plan(row_bytes=f * g.element_size())
    L.check(L.lib().gm_spmm_max_backward(C.byref(cs), C.byref(plan), _DT[g.dtype], _p(argmax.contiguous()), _p(g),
                                         f, _p(dx), _stream()), "gm_spmm_max_backward")
    return dx


# ---------------------------------------------------------------------------
# Generic message passing: select_path / propagate (message_passing.hpp:14-36,
# 176-258) over this library's gather, grouping and aggregation kernels.
# ---------------------------------------------------------------------------
EDGE_MATERIALIZE = "edge_materialize"
SEGMENT_FUSED = "segment_fused"


@dataclass
class MessageFns:
    """message(h_w, edge_attr, h_v) -> messages (edge-aligned) and
    update(h_v, aggregated) (message_passing.hpp:176-182). None = identity
    message (h_w) / update returning the aggregate."""
    message: Optional[object] = None
    update: Optional[object] = None


def select_path(e: EdgeIndex, needs_edge_callback: bool) -> str:
    """message_passing.hpp:31-36: an edge callback forces materialisation; the
    fused path needs a destination grouping (by_dst claim, CSC cache, or an
    undirected index's CSR cache)."""
    if needs_edge_callback:
        return EDGE_MATERIALIZE
    grouped = e.sort_order() == "by_dst" or e.has_csc_cache() or (e.is_undirected() and e.has_csr_cache())
    return SEGMENT_FUSED if grouped else EDGE_MATERIALIZE


def gather_rows(src: torch.Tensor, index, name: str = "gather_rows:") -> torch.Tensor:
    """tensor.hpp:499-530: out[i] = src[index[i]] after the bounds check of
    tensor.hpp:489-495 (std::out_of_range naming the first bad position)."""
    if src.dim() < 1:
        raise ValueError("gather_rows: rank >= 1 required")
    _same_device("gather_rows", src.device)
    n = src.shape[0]
    idx = index if isinstance(index, torch.Tensor) else torch.as_tensor(index)
    idx = idx.to(device=src.device)
    lib = L.lib()
    if idx.dtype == torch.int64:
        ws = torch.empty(64, dtype=torch.uint8, device=src.device)
        L.check(lib.gm_check_index_bounds(_p(idx), idx.numel(), n, name.encode(), _p(ws), _stream()), "bounds")
        idx = idx.to(torch.int32)
    idx = idx.contiguous()
    x = src.contiguous()
    f = 1
    for d in x.shape[1:]:
        f *= int(d)
    out = torch.empty((idx.numel(),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if idx.numel() and f:
        L.check(lib.gm_gather_rows(_DT[x.dtype], _p(x), f, _p(idx), idx.numel(), _p(out), _stream()),
                "gm_gather_rows")
    return out


def _entry_dst(grouping: CsrView) -> torch.Tensor:
    return grouping.entry_rows()[: grouping.num_entries()]


def propagate(e: EdgeIndex, h_src: torch.Tensor, h_dst: torch.Tensor, edge_attr: Optional[torch.Tensor],
              fns: MessageFns, agg: str, path: str, callback=None, edge_type_name: str = "") -> torch.Tensor:
    """message_passing.hpp:220-258: h'_v = update(h_v, agg_{w in N(v)} c(message(h_w, e_wv, h_v))).
    edge_materialize: messages in COO order, aggregated in ascending position
    per destination (aggregate's unsorted_scatter); segment_fused: messages in
    destination-grouped order (the CSC, or the exact grouping when an edge
    attribute meets an undirected index), sorted-segment aggregate. With an
    identity message and no edge attribute the fused path is one SpMM kernel
    (no E x F temporary)."""
    if h_src.shape[0] != e.num_src_nodes():
        raise ValueError("propagate: h_src rows != num_src_nodes")
    if h_dst.shape[0] != e.num_dst_nodes():
        raise ValueError("propagate: h_dst rows != num_dst_nodes")
    if edge_attr is not None and edge_attr.shape[0] != e.num_edges():
        raise ValueError("propagate: edge_attr rows != num_edges")
    _same_device("propagate", e.src().device, h_src, h_dst, edge_attr)
    if path == SEGMENT_FUSED and callback is not None:
        raise ValueError("propagate: edge callbacks require the edge_materialize path")
    if path not in (EDGE_MATERIALIZE, SEGMENT_FUSED):
        raise ValueError(f"propagate: unknown path {path}")
    message = fns.message or (lambda hw, ea, hv: hw)
    update = fns.update or (lambda hv, a: a)
    n_dst = e.num_dst_nodes()
    if path == EDGE_MATERIALIZE:
        hw = gather_rows(h_src, e.src())
        hv = gather_rows(h_dst, e.dst())
        m = message(hw, edge_attr, hv)
        if callback is not None:
            m = callback(m, edge_type_name)
        return update(h_dst, aggregate(m, e.dst(), n_dst, agg))
    if fns.message is None and edge_attr is None:
        return update(h_dst, neighbor_aggregate(e, h_src, agg))
    # the exact grouping on undirected indices: gathers the true in-neighbour
    # (see neighbor_aggregate), for every message function
    grouping = e._exact_dst_grouping() if e.is_undirected() else e.transpose_view()
    k = grouping.num_entries()
    hw = gather_rows(h_src, grouping.col[:k])
    grouped_dst = _entry_dst(grouping)
    hv = gather_rows(h_dst, grouped_dst)
    ea = gather_rows(edge_attr, grouping.perm[:k]) if edge_attr is not None else None
    m = message(hw, ea, hv)
    return update(h_dst, aggregate(m, grouped_dst, n_dst, agg))


def gcn_degrees(e: EdgeIndex, square: bool):
    """Effective degrees of gcn_norm (message_passing.hpp:437-463) from the FULL arrays,
    computed once per index (they depend only on the immutable COO arrays) and
    cached beside its CSR/CSC, like the reference caches its compressed views."""
    key = (bool(square), e.num_src_nodes(), e.num_dst_nodes())
    hit = e._cache.gcn_deg.get(key)
    if hit is not None:
        return hit
    dev = e.full_dst().device
    d_dst = torch.empty(e.num_dst_nodes(), dtype=torch.int32, device=dev)
    d_src = d_dst if square else torch.empty(e.num_src_nodes(), dtype=torch.int32, device=dev)
    L.check(L.lib().gm_gcn_degrees(_p(e.full_src()), _p(e.full_dst()), e.full_dst().numel(),
                                   e.num_src_nodes(), e.num_dst_nodes(), int(square), _p(d_src),
                                   _p(d_dst), _stream()), "gcn_degrees")
    e._cache.gcn_deg[key] = (d_src, d_dst)
    return d_src, d_dst


def gcn_aggregate(e: EdgeIndex, xw: torch.Tensor, bias: Optional[torch.Tensor] = None,
                  relu: bool = False) -> torch.Tensor:
    """GCN neighbour side after the transform (message_passing.hpp:490-495):
    with_self_loops + gcn_norm + spmm(sum), fused into one pass over e's CSC.
    bias / relu: layer_update's add(agg, bias) (:578) and the model's
    inter-layer relu (:637), applied in the same kernel's store epilogue."""
    if xw.shape[0] != e.num_src_nodes():
        raise ValueError("spmm: feature rows != num_src_nodes")
    square = e.num_src_nodes() == e.num_dst_nodes()
    d_src, d_dst = gcn_degrees(e, square)
    b = None
    if bias is not None:
        f = xw.shape[1] if xw.dim() == 2 else 1
        b = bias.to(device=xw.device, dtype=_acc_dtype(xw.dtype)).contiguous()
        if b.numel() != f:
            raise ValueError("layer_update: bias length != feature width")
    gcn = L.gm_gcn_norm(d_src.data_ptr(), d_dst.data_ptr(), int(square),
                        None if b is None else b.data_ptr(), int(bool(relu)))
    # with_self_loops builds a claim-less index, so its transpose_view is the CSC
    return _run_spmm(e.to_csc(), xw, "sum", gcn=gcn, num_rows=e.num_dst_nodes())


def gcn_layer(e: EdgeIndex, h: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor,
              relu: bool = False) -> torch.Tensor:
    """layer_forward for LayerKind::gcn (message_passing.hpp:490-499, 578), two
    launches of this library: the transform h @ W on the tcgen05 grouped GEMM
    (one group; fp32 operands take the fp32-accurate split route, the
    reference's matmul<float>), then the fused aggregate whose epilogue adds
    the bias (and the optional inter-layer relu)."""
    if h.dim() != 2 or h.shape[0] != e.num_src_nodes() or e.num_src_nodes() != e.num_dst_nodes():
        raise ValueError("layer_forward: square index matching h required")
    if weight.dim() != 2 or weight.shape[0] != h.shape[1]:
        raise ValueError("matmul: inner dimension mismatch")
    if h.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("gcn_layer: f32 or bf16 features")
    _same_device("gcn_layer", e.src().device, h, weight, bias)
    w = weight.to(h.dtype).unsqueeze(0)
    xw = segment_matmul(h, [0, h.shape[0]], w, out_dtype=h.dtype)
    return gcn_aggregate(e, xw, bias=bias, relu=relu)


def gcn_forward(e: EdgeIndex, x: torch.Tensor, layers: Sequence[tuple]) -> torch.Tensor:
    """Model::forward for a GCN stack (message_passing.hpp:631-641, no head):
    relu between layers, fused into each aggregate's epilogue.
    layers: [(weight, bias), ...]."""
    h = x
    for i, (w, b) in enumerate(layers):
        h = gcn_layer(e, h, w, b, relu=i + 1 < len(layers))
    return h


def aggregate(values: torch.Tensor, index: torch.Tensor, num_groups: int, kind: str) -> torch.Tensor:
    """aggregate.hpp:154-215 (sum/mean/max/min) for edge-level rows: groups are
    visited in ascending position, exactly the reference's scatter order."""
    if kind not in _KIND:
        raise ValueError(f"unknown aggregation kind: {kind}")
    _same_device("aggregate", values.device)
    index = index.to(device=values.device, dtype=torch.int64).contiguous()
    if values.shape[0] != index.numel():
        raise ValueError("aggregate: values rows != index length")
    lib = L.lib()
    ws = torch.empty(64, dtype=torch.uint8, device=index.device)
    L.check(lib.gm_check_index_bounds(_p(index), index.numel(), num_groups, b"aggregate:", _p(ws),
                                      _stream()), "bounds")
    positions = torch.arange(index.numel(), dtype=torch.int64, device=index.device)
    grouping = build_compressed(index, positions, num_groups, index.numel())
    x = values if values.dim() == 2 else values.reshape(-1, 1)
    out = _run_spmm(grouping, x, kind, num_rows=num_groups)
    return out if values.dim() == 2 else out.reshape(-1)


# ---------------------------------------------------------------------------
# Grouped GEMM
# ---------------------------------------------------------------------------

def segment_matmul(x: torch.Tensor, ptr: Sequence[int], weights: torch.Tensor,
                   out_dtype: Optional[torch.dtype] = None) -> torch.Tensor:
    """out[ptr[g]:ptr[g+1]] = x[ptr[g]:ptr[g+1]] @ weights[g] (hetero.hpp:134-157)
    on tcgen05 tensor cores with fp32 accumulation. bf16 operands: one bf16
    GEMM (bf16 output by default). fp32 operands (the reference's
    grouped_matmul<float>): fp32-accurate split-bf16 GEMM (gm_segment_matmul_f32),
    fp32 output."""
    if weights.dim() != 3:
        raise ValueError("grouped_matmul: weights must be [groups, F, F']")
    groups, k, n = weights.shape
    if len(ptr) != groups + 1:
        raise ValueError(f"grouped_matmul: group count mismatch ({len(ptr) - 1} inputs, {groups} weight slabs)")
    if x.dim() != 2 or x.shape[1] != k:
        raise ValueError("grouped_matmul: inner dimension mismatch")
    _same_device("grouped_matmul", x.device, weights)
    ptr = [int(p) for p in (ptr.tolist() if isinstance(ptr, torch.Tensor) else ptr)]
    if ptr[0] != 0 or any(b < a for a, b in zip(ptr, ptr[1:])):
        raise ValueError("grouped_matmul: segment offsets must start at 0 and be non-decreasing")
    rows = ptr[-1]
    if rows != x.shape[0]:
        raise ValueError(f"grouped_matmul: segment offsets cover {rows} rows, x has {x.shape[0]}")
    if x.dtype == torch.float32 and weights.dtype == torch.float32 and out_dtype in (None, torch.float32):
        xf, wf = x.contiguous(), weights.contiguous()
        out = torch.empty((rows, n), dtype=torch.float32, device=x.device)
        ptr_h = (C.c_int64 * (groups + 1))(*[int(p) for p in ptr])
        lib = L.lib()
        ws_bytes = lib.gm_segment_matmul_f32_workspace(rows, groups, k, n)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
        L.check(lib.gm_segment_matmul_f32(_p(xf), ptr_h, groups, k, n, _p(wf), _p(out), _p(ws), ws_bytes, _stream()),
                "gm_segment_matmul_f32")
        return out
    out_dtype = out_dtype or torch.bfloat16
    w = weights.to(torch.bfloat16).contiguous()
    packed = _packed_weights(w, groups, k, n)
    if x.dtype == torch.float32 and out_dtype == torch.float32 and k % 4 == 0:
        # fp32 activations: rounded to bf16 inside the GEMM kernel (x read once)
        xf = x.contiguous()
        if xf.data_ptr() % 16 == 0:
            out = torch.empty((rows, n), dtype=torch.float32, device=x.device)
            ptr_h = (C.c_int64 * (groups + 1))(*[int(p) for p in ptr])
            lib = L.lib()
            ws_bytes = lib.gm_segment_matmul_packed_workspace(rows, groups, k, n)
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
            L.check(lib.gm_segment_matmul_packed_xf32(_p(xf), ptr_h, groups, k, n, _p(packed), _p(out), _p(ws),
                                                      ws_bytes, _stream()), "gm_segment_matmul_packed_xf32")
            return out
    x = x.to(torch.bfloat16).contiguous()
    out = torch.empty((rows, n), dtype=out_dtype, device=x.device)
    ptr_h = (C.c_int64 * (groups + 1))(*[int(p) for p in ptr])
    lib = L.lib()
    ws_bytes = lib.gm_segment_matmul_packed_workspace(rows, groups, k, n)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
    L.check(lib.gm_segment_matmul_packed(_p(x), ptr_h, groups, k, n, _p(packed), _DT[out_dtype], _p(out), _p(ws),
                                         ws_bytes, _stream()), "gm_segment_matmul_packed")
    return out


def _packed_weights(w: torch.Tensor, groups: int, k: int, n: int) -> torch.Tensor:
    """K-major padded W^T for the tcgen05 kernel, packed once per weight tensor
    version and kept on the tensor (re-packed after any in-place update)."""
    hit = getattr(w, "_gm_packed", None)
    if hit is not None and hit[0] == w._version and hit[1] == (groups, k, n):
        return hit[2]
    lib = L.lib()
    packed = torch.empty(max(lib.gm_segment_matmul_packed_w_bytes(groups, k, n), 1), dtype=torch.uint8,
                         device=w.device)
    L.check(lib.gm_segment_matmul_pack_w(_p(w), groups, k, n, _p(packed), _stream()), "gm_segment_matmul_pack_w")
    w._gm_packed = (w._version, (groups, k, n), packed)
    return packed


def grouped_matmul(inputs: Sequence[torch.Tensor], weights: torch.Tensor,
                   out_dtype: Optional[torch.dtype] = None, out: Optional[Sequence[torch.Tensor]] = None):
    """List form of hetero.hpp:134-157 (validates like the reference): one
    gm_grouped_matmul launch reads every group's tensor in place and writes
    every group's output in place (per-group TMA maps; no concatenation).
    fp32 inputs and weights take the fp32-accurate route; otherwise bf16.
    out (optional): per-group destination tensors."""
    if weights.dim() != 3:
        raise ValueError("grouped_matmul: weights must be [groups, F, F']")
    groups, k, n = weights.shape
    if len(inputs) != groups:
        raise ValueError(f"grouped_matmul: group count mismatch ({len(inputs)} inputs, {groups} weight slabs)")
    for g, h in enumerate(inputs):
        if h.dim() != 2 or h.shape[1] != k:
            raise ValueError(f"grouped_matmul: group {g} inner dimension mismatch")
    _same_device("grouped_matmul", weights.device, *inputs, *(out or []))
    dev = weights.device
    x32 = all(h.dtype == torch.float32 for h in inputs)
    if x32 and weights.dtype == torch.float32 and out_dtype in (None, torch.float32):
        # the reference's grouped_matmul<float>: fp32-accurate split route
        xs, w = [h.contiguous() for h in inputs], weights.contiguous()
        odt, xdt, wdt = torch.float32, L.GM_F32, L.GM_F32
    elif x32 and out_dtype in (None, torch.float32) and k % 4 == 0:
        # fp32 activations x bf16 weights: rounded to bf16 inside the kernel
        xs, w = [h.contiguous() for h in inputs], weights.to(torch.bfloat16).contiguous()
        odt, xdt, wdt = torch.float32, L.GM_F32, L.GM_BF16
    else:
        xs = [h.to(torch.bfloat16).contiguous() for h in inputs]
        w = weights.to(torch.bfloat16).contiguous()
        odt, xdt, wdt = out_dtype or torch.bfloat16, L.GM_BF16, L.GM_BF16
    if out is None:
        outs = [torch.empty((h.shape[0], n), dtype=odt, device=dev) for h in xs]
    else:
        outs = list(out)
        for g, o in enumerate(outs):
            if tuple(o.shape) != (xs[g].shape[0], n) or o.dtype != odt or not o.is_contiguous():
                raise ValueError(f"grouped_matmul: out[{g}] must be a contiguous [{xs[g].shape[0]}, {n}] {odt}")
    rows = (C.c_int64 * groups)(*[int(h.shape[0]) for h in xs])
    xp = (C.c_void_p * groups)(*[h.data_ptr() for h in xs])
    op = (C.c_void_p * groups)(*[o.data_ptr() for o in outs])
    lib = L.lib()
    nb = lib.gm_grouped_matmul_workspace(rows, groups, k, n, xdt, wdt, _DT[odt])
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    L.check(lib.gm_grouped_matmul(xp, rows, groups, k, n, _p(w), xdt, wdt, op, _DT[odt], _p(ws), nb, _stream()),
            "gm_grouped_matmul")
    return outs
