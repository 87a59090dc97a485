"""ctypes binding of the C-ABI in include/graphmill_b200.h.

This is exactly the binding a maintainer of the reference would add on its
side of the boundary. It loads the in-tree
``libgraphmill_b200.so`` and fails loudly if it is missing: there is no CPU
fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# GM_LIB_PATH selects an alternative in-tree build (A/B kernel experiments only)
LIB_PATH = os.environ.get("GM_LIB_PATH") or os.path.join(_HERE, "libgraphmill_b200.so")

GM_OK = 0
GM_ERR_INVALID_ARGUMENT = 1
GM_ERR_OUT_OF_RANGE = 2
GM_ERR_CUDA = 3
GM_ERR_UNSUPPORTED = 4
GM_ERR_LOGIC = 5
GM_ERR_RUNTIME = 6
GM_ERR_NCCL = 7

GM_F32, GM_F64, GM_BF16 = 0, 1, 2
GM_SUM, GM_MEAN, GM_MAX, GM_MIN = 0, 1, 2, 3


class gm_csr(C.Structure):
    _fields_ = [
        ("num_rows", C.c_int64),
        ("num_cols", C.c_int64),
        ("nnz", C.c_int64),
        ("rowptr", C.c_void_p),
        ("col", C.c_void_p),
        ("perm", C.c_void_p),
    ]


class gm_spmm_plan(C.Structure):
    _fields_ = [
        ("num_windows", C.c_int64),
        ("window_edges", C.c_int64),
        ("num_heavy", C.c_int64),
        ("heavy_threshold", C.c_int64),
        ("win_row", C.c_void_p),
        ("heavy_rows", C.c_void_p),
        ("num_light_windows", C.c_int64),
        ("light_windows", C.c_void_p),
        ("src_class", C.c_void_p),
        ("l2_hot_bytes", C.c_int64),
        ("hot_edge_frac", C.c_float * 128),
    ]


class gm_gcn_norm(C.Structure):
    _fields_ = [("deg_src", C.c_void_p), ("deg_dst", C.c_void_p), ("self_loops", C.c_int),
                ("bias", C.c_void_p), ("relu", C.c_int)]


GM_MAX_PUSH = 8
GM_CARRY_NONE, GM_CARRY_START, GM_CARRY_CONTINUE, GM_CARRY_FINISH = 0, 1, 2, 3


class gm_spmm_epilogue(C.Structure):
    _fields_ = [
        ("carry", C.c_void_p),
        ("carry_mode", C.c_int32),
        ("n_push", C.c_int32),
        ("push_dst", C.c_void_p * GM_MAX_PUSH),
        ("push_row0", C.c_int64),
        ("push_mask", C.c_void_p),
    ]


GM_DIST_EXACT, GM_DIST_BLOCKED, GM_DIST_HALO = 0, 1, 2


class gm_dist_layout(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("mode", C.c_int),
        ("chunks", C.c_int32),
        ("shard_rows", C.c_int64),
        ("chunk_rows", C.c_int64),
        ("blocks", C.POINTER(gm_csr)),
        ("plans", C.POINTER(gm_spmm_plan)),
        ("mean_deg", C.c_void_p),
        ("halo_send_idx", C.c_void_p),
        ("halo_send_counts_host", C.POINTER(C.c_int64)),
        ("halo_recv_counts_host", C.POINTER(C.c_int64)),
    ]


# name -> (restype, argtypes); mirrors include/graphmill_b200.h one to one.
_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
SIGNATURES = {
    "gm_last_error": (C.c_char_p, []),
    "gm_version": (C.c_char_p, []),
    "gm_device_supported": (C.c_int, []),
    "gm_check_index_bounds": (C.c_int, [_P, _I64, _I64, C.c_char_p, _P, _P]),
    "gm_first_unsorted": (C.c_int, [_P, _I64, C.POINTER(C.c_int64), _P, _P]),
    "gm_degree": (C.c_int, [_P, _I64, _I64, _P, _P]),
    "gm_first_asymmetric_workspace": (C.c_size_t, [_I64]),
    "gm_first_asymmetric": (C.c_int, [_P, _P, _I64, _I64, C.POINTER(C.c_int64), _P, C.c_size_t, _P]),
    "gm_build_compressed_workspace": (C.c_size_t, [_I64, _I64]),
    "gm_build_compressed": (C.c_int, [_P, _P, _I64, _I64, _P, _P, _P, _P, C.c_size_t, _P]),
    "gm_permute_edge_values": (C.c_int, [C.c_int, _P, _P, _I64, _P, _P]),
    "gm_spmm_plan_bytes": (C.c_size_t, [_I64, _I64, _I64]),
    "gm_spmm_plan_build": (C.c_int, [C.POINTER(gm_csr), _P, C.c_size_t, C.POINTER(gm_spmm_plan), _P]),
    "gm_gcn_degrees": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, _P, _P, _P]),
    "gm_spmm": (C.c_int, [C.POINTER(gm_csr), C.POINTER(gm_spmm_plan), C.c_int, _P, _I64, _P,
                          C.POINTER(gm_gcn_norm), C.c_int, _P, _P, _P]),
    "gm_spmm_accumulate": (C.c_int, [C.POINTER(gm_csr), C.POINTER(gm_spmm_plan), C.c_int, _P, _I64, _P,
                                     C.c_int, _P, _P, _P, _P]),
    "gm_spmm_ex": (C.c_int, [C.POINTER(gm_csr), C.POINTER(gm_spmm_plan), C.c_int, _P, _I64, _P, C.c_int,
                             C.c_int32, _P, C.POINTER(gm_spmm_epilogue), _P, _P, _P]),
    "gm_ipc_handle_bytes": (C.c_size_t, []),
    "gm_ipc_get_handle": (C.c_int, [_P, _P]),
    "gm_ipc_open_handle": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "gm_ipc_close_handle": (C.c_int, [_P]),
    "gm_mark_columns": (C.c_int, [C.POINTER(gm_csr), _P, _P]),
    "gm_gather_rows": (C.c_int, [C.c_int, _P, _I64, _P, _I64, _P, _P]),
    "gm_csr_split_blocks_workspace": (C.c_size_t, [_I64, C.c_int32]),
    "gm_csr_split_blocks": (C.c_int, [C.POINTER(gm_csr), _P, _P, C.c_int32, _P, _P, _P, _P, C.c_size_t, _P]),
    "gm_scale_rows_div": (C.c_int, [C.c_int, _P, _I64, _I64, _P, _P, _P]),
    "gm_edge_dot": (C.c_int, [C.c_int, _P, _P, _I64, _P, _P, _I64, _P, _P]),
    "gm_csr_entry_rows": (C.c_int, [C.POINTER(gm_csr), _P, _P]),
    "gm_edge_dot_csc": (C.c_int, [C.c_int, C.POINTER(gm_csr), C.POINTER(gm_spmm_plan), _P, _P, _P, _I64, _P, _P]),
    "gm_source_view_workspace": (C.c_size_t, [_I64, _I64]),
    "gm_source_view": (C.c_int, [C.POINTER(gm_csr), _I64, _P, _P, _P, _P, C.c_size_t, _P]),
    "gm_spmm_max_backward": (C.c_int, [C.POINTER(gm_csr), C.POINTER(gm_spmm_plan), C.c_int, _P, _P, _I64, _P, _P]),
    "gm_hetero_combine": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, _P, _P, _I64, _I64, _P, _P]),
    "gm_segment_matmul_workspace": (C.c_size_t, [_I64, _I64, _I64, _I64]),
    "gm_segment_matmul": (C.c_int, [_P, C.POINTER(C.c_int64), _I64, _I64, _I64, _P, C.c_int, _P,
                                    _P, C.c_size_t, _P]),
    "gm_segment_matmul_packed_w_bytes": (C.c_size_t, [_I64, _I64, _I64]),
    "gm_segment_matmul_pack_w": (C.c_int, [_P, _I64, _I64, _I64, _P, _P]),
    "gm_segment_matmul_packed_workspace": (C.c_size_t, [_I64, _I64, _I64, _I64]),
    "gm_segment_matmul_packed": (C.c_int, [_P, C.POINTER(C.c_int64), _I64, _I64, _I64, _P, C.c_int, _P, _P,
                                           C.c_size_t, _P]),
    "gm_segment_matmul_packed_xf32": (C.c_int, [_P, C.POINTER(C.c_int64), _I64, _I64, _I64, _P, _P, _P, C.c_size_t,
                                                _P]),
    "gm_segment_matmul_f32_workspace": (C.c_size_t, [_I64, _I64, _I64, _I64]),
    "gm_segment_matmul_f32": (C.c_int, [_P, C.POINTER(C.c_int64), _I64, _I64, _I64, _P, _P, _P, C.c_size_t, _P]),
    "gm_grouped_matmul_workspace": (C.c_size_t, [C.POINTER(C.c_int64), _I64, _I64, _I64, C.c_int, C.c_int, C.c_int]),
    "gm_grouped_matmul": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_int64), _I64, _I64, _I64, _P, C.c_int,
                                    C.c_int, C.POINTER(C.c_void_p), C.c_int, _P, C.c_size_t, _P]),
    "gm_partition_rows_by_nnz": (C.c_int, [C.POINTER(C.c_int64), _I64, C.c_int32,
                                           C.POINTER(C.c_int64)]),
    "gm_nccl_unique_id": (C.c_int, [_P]),
    "gm_nccl_comm_init": (C.c_int, [C.c_int32, _P, C.c_int32, C.POINTER(C.c_void_p)]),
    "gm_nccl_comm_destroy": (C.c_int, [_P]),
    "gm_dist_spmm_workspace": (C.c_size_t, [C.POINTER(gm_dist_layout), C.c_int, _I64]),
    "gm_dist_spmm": (C.c_int, [C.POINTER(gm_dist_layout), C.c_int, _P, _I64, C.c_int, _P, _P, _P, C.c_size_t, _P, _P,
                               _P]),
    "gm_read_file_to_device": (C.c_int, [C.c_char_p, _I64, _P, _P, C.c_size_t, _P]),
    "gm_read_edge_pairs_workspace": (C.c_size_t, [C.c_size_t]),
    "gm_read_edge_pairs_to_device": (C.c_int, [C.c_char_p, _I64, _P, _P, _P, C.c_size_t, _P, C.c_size_t, _P]),
    "gm_synth_edges": (C.c_int, [C.c_int, _U64, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "gm_synth_edges_host": (None, [C.c_int, _U64, _I64, _I64, _I64, _I64, _P, _P]),
    "gm_synth_features": (C.c_int, [_U64, _I64, _I64, _I64, C.c_int, C.c_int, _P, _P]),
    "gm_synth_features_host": (None, [_U64, _I64, _I64, _I64, C.c_int, C.c_int, _P]),
    "gm_synth_weights": (C.c_int, [_U64, _I64, _I64, C.c_int, _P, _P]),
    "gm_synth_weights_host": (None, [_U64, _I64, _I64, C.c_int, _P]),
}


class GraphmillError(RuntimeError):
    pass


_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    cmd = ["make", "-C", os.path.join(_HERE, "csrc"), "-j8"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise GraphmillError("building libgraphmill_b200.so failed:\n" + (out.stderr or "")[-4000:])
    return LIB_PATH


def lib():
    """The loaded C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GraphmillError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, what: str = "") -> None:
    """Map a gm_status to the reference's exception types."""
    if status == GM_OK:
        return
    msg = lib().gm_last_error().decode()
    if status == GM_ERR_OUT_OF_RANGE:
        raise IndexError(msg)          # std::out_of_range
    if status == GM_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if status == GM_ERR_RUNTIME:
        raise RuntimeError(msg)        # std::runtime_error (dataset IO)
    raise GraphmillError(f"{what}: status {status}: {msg}")
