"""Heterogeneous (RGCN-shaped) layer on B200: the reference's
``to_hetero(sage)`` + ``hetero_propagate`` with ``InterCombine::sum``
(hetero.hpp:217-365), composed from the hot-path kernels:

  1. per edge type (sorted canonical order, hetero.hpp:294-300):
       agg_et = spmm(e_et, h[src_type], mean)               exact fp32 (gm_spmm)
  2. neighbour projection for ALL edge types at once:
       P = segment_matmul(cat(agg_et), stack(w_neigh_et))  tcgen05 grouped GEMM
     (message_passing.hpp:520, one matmul per edge type in the reference)
  3. self projection for ALL node types at once:
       S = grouped_matmul([h_nt], stack(w_self_nt))        tcgen05 grouped GEMM,
     every h_nt read in place (per-group TMA maps)
     (layer_update message_passing.hpp:579-580, one matmul per node type)
  4. out_nt = ((sum_et P_et) + S_nt) + bias_nt              gm_hetero_combine,
     in the reference's add order (hetero.hpp:338-343, :362)

Steps 1 and 4 are bit-exact; 2 and 3 run bf16 operands with fp32
accumulation (the segment_matmul tolerance, tests/test_gpu_gemm.py).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Tuple

import torch

from . import _lib as L
from .graphmill import EdgeIndex, _stream, grouped_matmul, segment_matmul, spmm

EdgeKey = Tuple[str, str, str]  # (src, rel, dst) — EdgeType


def canonical(et: EdgeKey) -> str:
    """EdgeType::canonical (hetero.hpp:16-22): src__rel__dst."""
    return f"{et[0]}__{et[1]}__{et[2]}"


def hetero_sage_layer(edges: Dict[EdgeKey, EdgeIndex], h: Dict[str, torch.Tensor],
                      w_neigh: Dict[EdgeKey, torch.Tensor], w_self: Dict[str, torch.Tensor],
                      bias: Dict[str, torch.Tensor]) -> Dict[str, torch.Tensor]:
    node_types = sorted(h)                       # std::map order
    edge_types = sorted(edges, key=canonical)    # EdgeType::operator< (canonical)
    for nt in node_types:
        if nt not in w_self or nt not in bias:
            raise ValueError(f"hetero_propagate: model lacks update params for type {nt}")
    for et in edge_types:
        if et[0] not in h or et[2] not in h:
            raise ValueError(f"hetero_propagate: missing node type {et[0] if et[0] not in h else et[2]}")
        if et not in w_neigh:
            raise ValueError(f"hetero_propagate: model lacks a replica for edge type {canonical(et)}")
    f_out = next(iter(w_self.values())).shape[1]
    f_in = next(iter(h.values())).shape[1]
    for nt in node_types:  # one feature width for every node type (the stacked weights' inner dimension)
        if h[nt].dim() != 2 or h[nt].shape[1] != f_in or w_self[nt].shape[0] != f_in:
            raise ValueError(f"hetero_propagate: node type {nt} feature width differs from {f_in}")
    dev = next(iter(h.values())).device

    # 1. per-edge-type mean aggregation (exact), written straight into the
    #    segments of the grouped GEMM's input (no concatenation copy)
    ptr = [0]
    for et in edge_types:
        ptr.append(ptr[-1] + edges[et].num_dst_nodes())
    agg_all = torch.empty(ptr[-1], f_in, dtype=next(iter(h.values())).dtype, device=dev)
    for i, et in enumerate(edge_types):
        spmm(edges[et], h[et[0]], None, "mean", out=agg_all[ptr[i]:ptr[i + 1]])
    # 2. one grouped GEMM over edge types (tcgen05)
    parts_by_dst: Dict[str, list] = {nt: [] for nt in node_types}
    if edge_types:
        proj = segment_matmul(agg_all, ptr, torch.stack([w_neigh[et] for et in edge_types]),
                              out_dtype=torch.float32)
        for i, et in enumerate(edge_types):
            parts_by_dst[et[2]].append(proj[ptr[i]:ptr[i + 1]])
    # 3. one grouped GEMM over node types (tcgen05), reading every node type's
    #    features in place (per-group TMA maps, no concatenation)
    selfp = grouped_matmul([h[nt] for nt in node_types], torch.stack([w_self[nt] for nt in node_types]),
                           out_dtype=torch.float32)
    # 4. combine in the reference's order
    out = {}
    lib = L.lib()
    for i, nt in enumerate(node_types):
        rows = h[nt].shape[0]
        o = torch.empty(rows, f_out, dtype=torch.float32, device=dev)
        parts = [p.contiguous() for p in parts_by_dst[nt]]
        arr = (C.c_void_p * max(1, len(parts)))(*[p.data_ptr() for p in parts])
        s = selfp[i]
        b = bias[nt].to(torch.float32).contiguous()
        L.check(lib.gm_hetero_combine(arr, len(parts), C.c_void_p(s.data_ptr()), C.c_void_p(b.data_ptr()),
                                      rows, f_out, C.c_void_p(o.data_ptr()), _stream()), "gm_hetero_combine")
        out[nt] = o
    return out
