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
