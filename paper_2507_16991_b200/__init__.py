"""graphmill-b200: B200-native (sm_100a) CSR message-passing hot path.

The compute lives in libgraphmill_b200.so (C-ABI, include/graphmill_b200.h);
`graphmill` mirrors the reference engine's operator API over it.
"""
from . import _lib  # noqa: F401
from .graphmill import (  # noqa: F401
    EDGE_MATERIALIZE, SEGMENT_FUSED, MessageFns, gather_rows, propagate, select_path, CsrView, EdgeIndex, aggregate, build_compressed, gcn_aggregate, gcn_forward, gcn_layer, grouped_matmul,
    neighbor_aggregate, neighbor_aggregate_backward, segment_matmul, spmm, spmm_backward)

__all__ = ["EDGE_MATERIALIZE", "SEGMENT_FUSED", "MessageFns", "gather_rows", "propagate", "select_path", "CsrView", "EdgeIndex", "aggregate", "build_compressed", "gcn_aggregate", "gcn_forward", "gcn_layer",
           "grouped_matmul", "neighbor_aggregate", "neighbor_aggregate_backward", "segment_matmul", "spmm", "spmm_backward"]
