"""Device ingestion of the reference's on-disk dataset format (SURVEY.md §8f
rank 4). The golden datasets under tests/golden/dataset_{f32,f64} were written
by the REFERENCE's own save_dataset (oracle/ref_dataset_gen.cpp, built by
`make -C oracle ref-dataset`; regenerate with tests/make_golden.py --dataset),
so the loader is pinned to the reference writer's bytes."""
import json
import os
import shutil

import numpy as np
import pytest
import torch

import paper_2507_16991_b200.dataset as ds
from paper_2507_16991_b200 import _lib as L

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _expect(d):
    man = json.load(open(os.path.join(d, "manifest.json")))
    return man


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dataset_f32", "dataset_f64"])
def test_load_reference_written_dataset(name):
    d = os.path.join(GOLD, name)
    man = _expect(d)
    got = ds.load_dataset(d)
    for n in man["node_types"]:
        tok = "f32" if n["dtype"] == "float32" else "f64"
        want = np.fromfile(os.path.join(d, f"node_{n['name']}.{tok}.bin"),
                           dtype=np.float32 if tok == "f32" else np.float64).reshape(n["count"], n["feature_width"])
        assert got.features[n["name"]].cpu().numpy().tobytes() == want.tobytes()
        if n["has_time"]:
            t = np.fromfile(os.path.join(d, f"node_{n['name']}.time.i64.bin"), dtype=np.int64)
            assert np.array_equal(got.node_times[n["name"]].cpu().numpy(), t)
    for e in man["edge_types"]:
        c = f"{e['src']}__{e['rel']}__{e['dst']}"
        pairs = np.fromfile(os.path.join(d, f"edge_{c}.u64.bin"), dtype=np.uint64).reshape(-1, 2).astype(np.int64)
        g = got.edges[c]
        assert g.num_edges() == e["edge_count"]
        assert np.array_equal(g.src().cpu().numpy(), pairs[:, 0])
        assert np.array_equal(g.dst().cpu().numpy(), pairs[:, 1])
        if e["has_time"]:
            t = np.fromfile(os.path.join(d, f"edge_{c}.time.i64.bin"), dtype=np.int64)
            assert np.array_equal(got.edge_times[c].cpu().numpy(), t)


@pytest.mark.gpu
def test_byte_length_and_bounds_errors(tmp_path):
    d = tmp_path / "ds"
    shutil.copytree(os.path.join(GOLD, "dataset_f32"), d)
    f = d / "edge_paper__cites__paper.u64.bin"
    raw = f.read_bytes()
    f.write_bytes(raw[:-8])
    with pytest.raises(RuntimeError, match=r"holds 2504 bytes, manifest requires 2512"):
        ds.load_dataset(str(d))
    # an out-of-range id is caught by the device EdgeIndex bounds check
    arr = np.frombuffer(raw, dtype=np.uint64).copy()
    arr[7] = 10_000  # pair 3's dst
    f.write_bytes(arr.tobytes())
    with pytest.raises(IndexError, match=r"EdgeIndex: dst index 10000 at position 3 outside \[0, 53\)"):
        ds.load_dataset(str(d))


@pytest.mark.gpu
def test_multi_chunk_pipeline(tmp_path, monkeypatch):
    """Many staging chunks (1 MiB staging) over a 24 MB pairs file and a 12 MB feature file."""
    monkeypatch.setattr(ds, "STAGING_BYTES", 1 << 20)
    rng = np.random.default_rng(3)
    n, e, f = 300_001, 1_500_007, 10
    d = tmp_path / "big"
    d.mkdir()
    x = rng.standard_normal((n, f)).astype(np.float32)
    x.tofile(d / "node_v.f32.bin")
    pairs = rng.integers(0, n, size=(e, 2)).astype(np.uint64)
    pairs.tofile(d / "edge_v__r__v.u64.bin")
    json.dump({"format": "graphmill.dataset", "version": 1,
               "node_types": [{"name": "v", "count": n, "feature_width": f, "dtype": "float32", "has_time": False}],
               "edge_types": [{"src": "v", "rel": "r", "dst": "v", "edge_count": e, "has_time": False}]},
              open(d / "manifest.json", "w"))
    got = ds.load_dataset(str(d))
    assert got.features["v"].cpu().numpy().tobytes() == x.tobytes()
    g = got.edges["v__r__v"]
    assert np.array_equal(g.src().cpu().numpy(), pairs[:, 0].astype(np.int64))
    assert np.array_equal(g.dst().cpu().numpy(), pairs[:, 1].astype(np.int64))


def test_manifest_validation_messages(tmp_path):
    """read_manifest's checks (dataset_io.cpp:45-93) run on the host, no GPU needed."""
    with pytest.raises(RuntimeError, match="dataset: missing manifest"):
        ds.read_manifest(str(tmp_path))
    (tmp_path / "manifest.json").write_text("{not json")
    with pytest.raises(RuntimeError, match="dataset: unparseable manifest"):
        ds.read_manifest(str(tmp_path))
    (tmp_path / "manifest.json").write_text(json.dumps({"format": "nope", "version": 1}))
    with pytest.raises(RuntimeError, match="corrupt magic .* \\(expected format 'graphmill.dataset'\\)"):
        ds.read_manifest(str(tmp_path))
    (tmp_path / "manifest.json").write_text(json.dumps({"format": "graphmill.dataset", "version": 2}))
    with pytest.raises(RuntimeError, match="unsupported version"):
        ds.read_manifest(str(tmp_path))
    bad = {"format": "graphmill.dataset", "version": 1,
           "node_types": [{"name": "a", "count": 1, "feature_width": 1, "dtype": "float16", "has_time": False}],
           "edge_types": []}
    (tmp_path / "manifest.json").write_text(json.dumps(bad))
    with pytest.raises(ValueError, match="unknown dtype: float16"):
        ds.read_manifest(str(tmp_path))
    man = ds.read_manifest(os.path.join(GOLD, "dataset_f64"))
    assert [n["name"] for n in man["node_types"]] == ["author", "paper"]


@pytest.mark.gpu
def test_int64_feature_column(tmp_path):
    """An int64 node feature column (dtype "int64", file token i64, 8-byte
    elements: dataset_io.hpp:44-50, dataset_io.cpp:289-305) loads as int64."""
    rng = np.random.default_rng(11)
    n, f, e = 1000, 3, 5000
    d = tmp_path / "i64"
    d.mkdir()
    x = rng.integers(-(1 << 40), 1 << 40, size=(n, f)).astype(np.int64)
    x.tofile(d / "node_v.i64.bin")
    pairs = rng.integers(0, n, size=(e, 2)).astype(np.uint64)
    pairs.tofile(d / "edge_v__r__v.u64.bin")
    json.dump({"format": "graphmill.dataset", "version": 1,
               "node_types": [{"name": "v", "count": n, "feature_width": f, "dtype": "int64", "has_time": False}],
               "edge_types": [{"src": "v", "rel": "r", "dst": "v", "edge_count": e, "has_time": False}]},
              open(d / "manifest.json", "w"))
    got = ds.load_dataset(str(d))
    assert got.features["v"].dtype == torch.int64
    assert np.array_equal(got.features["v"].cpu().numpy(), x)
