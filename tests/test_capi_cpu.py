"""CPU suite for the drop-in boundary: the C-ABI library loads here (no GPU),
exports every symbol include/graphmill_b200.h declares, and its host-side
logic (synthetic generators, partitioner, error plumbing) is correct."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2507_16991_b200 import _lib as L
import refrng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "graphmill_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"GM_API\s+[\w\s\*]+?\b(gm_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("gm_build_compressed", "gm_spmm", "gm_spmm_plan_build", "gm_segment_matmul",
                 "gm_check_index_bounds", "gm_gcn_degrees", "gm_partition_rows_by_nnz"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes signature table covers the header one to one
    assert set(declared_symbols()) == set(L.SIGNATURES)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {L.LIB_PATH} 2>/dev/null").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_error_plumbing():
    lib = L.lib()
    assert b"sm_100a" in lib.gm_version()
    # a validation failure sets the thread-local message without touching CUDA
    st = lib.gm_build_compressed(None, None, -1, 3, None, None, None, None, 0, None)
    assert st == L.GM_ERR_INVALID_ARGUMENT
    assert b"negative size" in lib.gm_last_error()
    with pytest.raises(ValueError, match="negative size"):
        L.check(st)


def test_segment_matmul_argument_validation_without_cuda():
    # argument checks run before any device work: safe on a CPU-only host
    import ctypes as C
    lib = L.lib()
    ptr = (C.c_int64 * 2)(0, 8)
    fake = C.c_void_p(16)  # never dereferenced: validation fails first
    st = lib.gm_segment_matmul_packed_xf32(fake, ptr, 1, 6, 8, fake, fake, None, 0, None)
    assert st == L.GM_ERR_INVALID_ARGUMENT
    assert b"k % 4" in lib.gm_last_error()
    st = lib.gm_segment_matmul_packed_xf32(fake, ptr, 1, 8, 8, None, fake, None, 0, None)
    assert st == L.GM_ERR_INVALID_ARGUMENT and b"null packed weights" in lib.gm_last_error()
    st = lib.gm_segment_matmul_f32(fake, ptr, 1, 0, 8, fake, fake, None, 0, None)
    assert st == L.GM_ERR_INVALID_ARGUMENT and b"K and N must be positive" in lib.gm_last_error()


def test_host_uniform_generator_matches_reference_rng():
    # edge i draws next_below from Stream(derive(seed, "src"/"dst", i)) (random.hpp)
    lib = L.lib()
    seed, n_src, n_dst, count = 77, 1000, 37, 64
    src = np.zeros(count, np.int64)
    dst = np.zeros(count, np.int64)
    lib.gm_synth_edges_host(0, seed, 5, count, n_src, n_dst, src.ctypes.data, dst.ctypes.data)
    for i in range(count):
        assert src[i] == refrng.Stream(refrng.derive(seed, 0x737263, 5 + i)).next_below(n_src)
        assert dst[i] == refrng.Stream(refrng.derive(seed, 0x647374, 5 + i)).next_below(n_dst)


def test_host_features_match_rand_uniform_per_row():
    lib = L.lib()
    x = np.zeros((3, 4), np.float64)
    lib.gm_synth_features_host(9, 10, 3, 4, 0, L.GM_F64, x.ctypes.data)
    for r in range(3):
        s = refrng.Stream(refrng.derive(9, 0x66656174, 10 + r))
        assert list(x[r]) == [s.next_real(-1.0, 1.0) for _ in range(4)]


def test_powerlaw_generator_is_skewed_and_in_range():
    lib = L.lib()
    n, e = 20000, 200000
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    lib.gm_synth_edges_host(1, 3, 0, e, n, n, src.ctypes.data, dst.ctypes.data)
    assert src.min() >= 0 and src.max() < n and dst.min() >= 0 and dst.max() < n
    deg = np.bincount(dst, minlength=n)
    # Chung-Lu alpha = 0.5: expected max degree ~ E * 0.5 / sqrt(N) = 707
    assert 400 < deg.max() < 1100
    assert deg.min() >= 1 or (deg == 0).mean() < 0.01


def test_bf16_host_rounding_is_rne():
    lib = L.lib()
    x32 = np.zeros((64, 8), np.float32)
    xb = np.zeros((64, 8), np.uint16)
    lib.gm_synth_features_host(4, 0, 64, 8, 0, L.GM_F32, x32.ctypes.data)
    lib.gm_synth_features_host(4, 0, 64, 8, 0, L.GM_BF16, xb.ctypes.data)
    u = x32.view(np.uint32).astype(np.uint64)
    want = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(xb, want)


def test_partition_rows_by_nnz():
    lib = L.lib()
    deg = np.array([5, 0, 0, 100, 1, 1, 1, 1, 50, 0], np.int64)
    rowptr = np.concatenate([[0], np.cumsum(deg)])
    for parts in (1, 2, 3, 4, 8):
        cuts = np.zeros(parts + 1, np.int64)
        st = lib.gm_partition_rows_by_nnz(rowptr.ctypes.data_as(C.POINTER(C.c_int64)), deg.size, parts,
                                          cuts.ctypes.data_as(C.POINTER(C.c_int64)))
        assert st == 0
        assert cuts[0] == 0 and cuts[-1] == deg.size and np.all(np.diff(cuts) >= 0)
        for p in range(1, parts):
            target = -(-rowptr[-1] * p // parts)
            assert cuts[p] == min(np.searchsorted(rowptr, target, "left"), deg.size) or cuts[p] == cuts[p - 1]


def test_host_tensors_rejected_before_any_kernel_call():
    """The Python mirror refuses host tensors (they would reach the kernels as
    host pointers) with a ValueError, before the library is called."""
    import pytest
    import torch
    import paper_2507_16991_b200 as gm
    x = torch.zeros(4, 8)
    w = torch.zeros(1, 8, 8)
    with pytest.raises(ValueError, match="CUDA tensors required"):
        gm.segment_matmul(x, [0, 4], w)
    with pytest.raises(ValueError, match="CUDA tensors required"):
        gm.grouped_matmul([x], w)
    with pytest.raises(ValueError, match="CUDA tensors required"):
        gm.gather_rows(x, torch.tensor([0, 1]))
    with pytest.raises(ValueError, match="CUDA tensors required"):
        gm.aggregate(x, torch.tensor([0, 1, 1, 0]), 2, "sum")
