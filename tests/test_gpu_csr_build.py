"""build_compressed (edge_index.cpp:45-62) on B200 against the oracle
restatement (itself pinned to the reference, tests/test_oracle.py), across the
shapes that select each route of gm_build_compressed:

* the LSD radix sort (csr_radix.cuh, default): 1, 2 and 3 passes of up to
  11-bit digits;
* the bucketed stable sort (csr_bucket.cuh, GM_CSR_ALGO=bucket): many rows, power-law hub rows
  longer than a whole bucket (single-row buckets), few rows with millions of
  entries, keys confined to a narrow row band, duplicate edges;
* the scatter + per-row sort fallback (more buckets than fit shared memory).

Bar: rowptr, col, perm bit-identical.
"""
import numpy as np
import pytest
import torch

import paper_2507_16991_b200 as gm
from paper_2507_16991_b200 import _lib as L
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


def synth(kind, n_rows, n_cols, e, seed):
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    L.lib().gm_synth_edges_host(kind, seed, 0, e, n_cols, n_rows, src.ctypes.data, dst.ctypes.data)
    return src, dst


def check(keys, values, n_rows):
    got = gm.build_compressed(torch.from_numpy(keys).cuda(), torch.from_numpy(values).cuda(), n_rows)
    rp, col, perm = got.to_host()
    w_rp, w_col, w_perm = Oracle().build_compressed(keys, values, n_rows)
    assert np.array_equal(rp.numpy(), w_rp), "rowptr"
    assert np.array_equal(perm.numpy(), w_perm), "perm"
    assert np.array_equal(col.numpy(), w_col), "col"


@pytest.mark.parametrize("kind,n,e", [
    (0, 1000, 5_000),           # uniform, one bucket of rows
    (1, 50_000, 3_000_000),     # power-law, hubs of ~20K entries
    (1, 2_000, 4_000_000),      # power-law over few rows: hubs > one bucket (131,072) -> single-row buckets
    (0, 4_000_000, 6_000_000),  # many rows (1,954 row buckets)
    (1, 300_000, 12_000_000),   # many entry-count cuts
    (1, 4_000_000, 9_000_000),  # 22-bit keys: two 11-bit LSD passes
    (0, 40_000_000, 1_500_000), # 26-bit keys: three 9-bit passes, mostly empty rows
    (0, 1000, 5001),            # odd edge counts: the TMA scatter's tail element
    (1, 70_000, 1_234_567),
    (0, 9, 1),
])
def test_bucketed_build_bit_exact(kind, n, e):
    src, dst = synth(kind, n, n, e, seed=n + e)
    check(dst, src, n)


def test_few_rows_millions_of_entries():
    rng = np.random.default_rng(1)
    keys = rng.integers(0, 3, 2_500_000)
    vals = rng.integers(0, 1 << 30, keys.size)
    check(keys, vals, 3)


def test_narrow_band_and_duplicates():
    rng = np.random.default_rng(2)
    keys = rng.integers(7_000, 7_010, 400_000)  # all entries in 10 rows of a 20K-row view
    vals = np.repeat(rng.integers(0, 50, 200_000), 2)  # duplicate (key, value) pairs are legal
    check(keys, vals, 20_000)


def test_single_entry_and_tail_tile():
    check(np.array([5]), np.array([9]), 6)
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 100, 8192 * 3 + 17)  # a partial last tile
    check(keys, rng.integers(0, 1000, keys.size), 100)


def test_fallback_route_when_buckets_exceed_shared_memory():
    # 9M rows -> > 4096 row buckets: the scatter + per-row sort route
    src, dst = synth(1, 9_000_000, 9_000_000, 3_000_000, seed=4)
    check(dst, src, 9_000_000)


def test_build_is_deterministic_across_calls():
    src, dst = synth(1, 100_000, 100_000, 5_000_000, seed=5)
    k, v = torch.from_numpy(dst).cuda(), torch.from_numpy(src).cuda()
    a = gm.build_compressed(k, v, 100_000)
    b = gm.build_compressed(k, v, 100_000)
    assert torch.equal(a.perm, b.perm) and torch.equal(a.col, b.col) and torch.equal(a.rowptr, b.rowptr)
