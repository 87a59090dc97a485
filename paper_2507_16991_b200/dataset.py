"""Dataset ingestion straight to the device.

Mirrors the reference's `load_dataset(dir)` (dataset_io.hpp:114-116,
dataset_io.cpp:295-341) over its on-disk layout (dataset_io.hpp:14-20,
manifest read_manifest dataset_io.cpp:45-93): node feature matrices and
timestamps land in device tensors, every edge type's (src, dst) u64 pairs are
split into device int64 arrays by `gm_read_edge_pairs_to_device` and wrapped in
a device `EdgeIndex` (bounds verified on the device, as the reference's
EdgeIndex constructor does). File reads overlap host->device copies through a
pinned double buffer; the host never materialises the COO arrays.

Errors keep the reference's types and texts: std::runtime_error -> RuntimeError
("dataset: missing manifest ...", "dataset: corrupt magic in ...",
"dataset: <file> holds X bytes, manifest requires Y", ...),
std::invalid_argument -> ValueError ("unknown dtype: ...").
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Dict, Optional

import torch

from . import _lib as L
from .graphmill import EdgeIndex, _p, _stream

FORMAT = "graphmill.dataset"   # dataset_io.hpp:22
VERSION = 1                    # dataset_io.hpp:23
# dtype -> (torch dtype, file token): dataset_io.hpp:44-50; int64 columns are
# 8-byte elements (dataset_io.cpp:289-291 sizes every non-f32 dtype as 8 bytes)
_DTYPES = {"float32": (torch.float32, "f32"), "float64": (torch.float64, "f64"), "int64": (torch.int64, "i64")}
STAGING_BYTES = 64 << 20


@dataclass
class DeviceDataset:
    """What load_dataset serves, resident in HBM: per node type the feature
    matrix [count, width] (and optional int64 timestamps), per edge type
    (canonical src__rel__dst) an EdgeIndex (and optional int64 timestamps)."""

    features: Dict[str, torch.Tensor] = field(default_factory=dict)
    node_times: Dict[str, torch.Tensor] = field(default_factory=dict)
    edges: Dict[str, EdgeIndex] = field(default_factory=dict)
    edge_times: Dict[str, torch.Tensor] = field(default_factory=dict)
    manifest: dict = field(default_factory=dict)


def read_manifest(path_dir: str) -> dict:
    """dataset_io.cpp:45-93 (validation order and messages)."""
    path = os.path.join(path_dir, "manifest.json")
    if not os.path.exists(path):
        raise RuntimeError(f"dataset: missing manifest {path}")
    try:
        with open(path) as fh:
            j = json.load(fh)
    except Exception as ex:  # noqa: BLE001 - the reference wraps any parse error
        raise RuntimeError(f"dataset: unparseable manifest {path}: {ex}") from None
    if j.get("format") != FORMAT:
        raise RuntimeError(f"dataset: corrupt magic in {path} (expected format '{FORMAT}')")
    if j.get("version") != VERSION:
        raise RuntimeError(f"dataset: unsupported version in {path}")
    for n in j["node_types"]:
        if n["dtype"] not in _DTYPES:
            raise ValueError(f"unknown dtype: {n['dtype']}")
        if n["count"] < 0 or n["feature_width"] < 0:
            raise RuntimeError(f"dataset: negative extent for node type {n['name']}")
    for e in j["edge_types"]:
        if e["edge_count"] < 0:
            raise RuntimeError(f"dataset: negative edge count for {e['src']}__{e['rel']}__{e['dst']}")
    return j


class _Staging:
    def __init__(self, device, nbytes=STAGING_BYTES):
        self.host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        wsb = L.lib().gm_read_edge_pairs_workspace(nbytes)
        self.dev = torch.empty(max(wsb, 1), dtype=torch.uint8, device=device)
        self.nbytes, self.ws_bytes = nbytes, wsb


def _read(path: str, nbytes: int, out: torch.Tensor, stg: _Staging):
    L.check(L.lib().gm_read_file_to_device(path.encode(), nbytes, _p(out), _p(stg.host), stg.nbytes, _stream()),
            "gm_read_file_to_device")


def load_dataset(path_dir: str, device: str | torch.device = "cuda") -> DeviceDataset:
    """load_dataset (dataset_io.cpp:295-341) into device memory."""
    man = read_manifest(path_dir)
    out = DeviceDataset(manifest=man)
    stg = _Staging(device)
    counts = {}
    for n in man["node_types"]:
        name, cnt, width = n["name"], int(n["count"]), int(n["feature_width"])
        tdtype, token = _DTYPES[n["dtype"]]
        feat = torch.empty(cnt, width, dtype=tdtype, device=device)
        _read(os.path.join(path_dir, f"node_{name}.{token}.bin"), feat.numel() * feat.element_size(), feat, stg)
        out.features[name] = feat
        if n["has_time"]:
            t = torch.empty(cnt, dtype=torch.int64, device=device)
            _read(os.path.join(path_dir, f"node_{name}.time.i64.bin"), cnt * 8, t, stg)
            out.node_times[name] = t
        counts[name] = cnt
    lib = L.lib()
    for e in man["edge_types"]:
        canon = f"{e['src']}__{e['rel']}__{e['dst']}"
        if e["src"] not in counts or e["dst"] not in counts:
            raise RuntimeError(f"dataset: edge type {canon} references unknown node types")
        ne = int(e["edge_count"])
        src = torch.empty(ne, dtype=torch.int64, device=device)
        dst = torch.empty(ne, dtype=torch.int64, device=device)
        path = os.path.join(path_dir, f"edge_{canon}.u64.bin")
        L.check(lib.gm_read_edge_pairs_to_device(path.encode(), ne, _p(src), _p(dst), _p(stg.host), stg.nbytes,
                                                 _p(stg.dev), stg.ws_bytes, _stream()), "gm_read_edge_pairs_to_device")
        out.edges[canon] = EdgeIndex(src, dst, counts[e["src"]], counts[e["dst"]], device=device)
        if e["has_time"]:
            t = torch.empty(ne, dtype=torch.int64, device=device)
            _read(os.path.join(path_dir, f"edge_{canon}.time.i64.bin"), ne * 8, t, stg)
            out.edge_times[canon] = t
    return out
