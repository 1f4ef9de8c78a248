"""Native readers of the reference's capture formats (csrc/pf_ingest.cu): TB32 blobs
(tensorio.py:40-64) and binary PLY points (ply.py:80-139), pinned to what the reference's own
load_bundle returned for a bundle written by its save_bundle (tests/golden/bundle_tiny + .npz),
plus the reference's error cases. Host code: runs without a GPU.
"""

import os
import struct

import numpy as np
import pytest

from paper_2511_03126_b200 import ingest
from paper_2511_03126_b200.errors import BundleLoadError, BundleStructureError

HERE = os.path.dirname(os.path.abspath(__file__))
BUNDLE = os.path.join(HERE, "golden", "bundle_tiny")


def test_tb32_and_ply_match_reference_load(golden):
    g = golden("bundle_tiny")
    for j in range(3):
        np.testing.assert_array_equal(ingest.read_tensor(os.path.join(BUNDLE, f"views/{j}/depth.f32")), g["depth"][j])
        np.testing.assert_array_equal(ingest.read_tensor(os.path.join(BUNDLE, f"views/{j}/feat.f32")), g["features"][j])
    pos, col = ingest.read_ply_points(os.path.join(BUNDLE, "cloud.ply"))
    np.testing.assert_array_equal(pos, g["positions"])
    np.testing.assert_array_equal(col, g["colors"])
    assert ingest.png_size(os.path.join(BUNDLE, "views/0/image.png")) == g["depth"][0].shape


def _blob(path, rank, dims, payload):
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sI4H", b"TB32", rank, *dims))
        fh.write(payload)


def test_tb32_errors(tmp_path):
    with pytest.raises(BundleLoadError, match="missing tensor blob"):
        ingest.read_tensor(tmp_path / "nope.f32")
    p = tmp_path / "a.f32"
    p.write_bytes(b"TB3")
    with pytest.raises(BundleStructureError, match="truncated before header"):
        ingest.read_tensor(p)
    _blob(p, 2, (2, 3, 0, 0), np.zeros(6, "<f4").tobytes())
    assert ingest.read_tensor(p).shape == (2, 3)
    _blob(p, 2, (2, 3, 0, 0), np.zeros(5, "<f4").tobytes())
    with pytest.raises(BundleStructureError, match="payload is 20 bytes, expected 24"):
        ingest.read_tensor(p)
    _blob(p, 5, (2, 3, 0, 0), b"")
    with pytest.raises(BundleStructureError, match="bad tensor rank"):
        ingest.read_tensor(p)
    _blob(p, 2, (2, 0, 0, 0), b"")
    with pytest.raises(BundleStructureError, match="inconsistent dims"):
        ingest.read_tensor(p)
    _blob(p, 1, (4, 7, 0, 0), b"")
    with pytest.raises(BundleStructureError, match="inconsistent dims"):
        ingest.read_tensor(p)
    p.write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(BundleStructureError, match="bad tensor magic"):
        ingest.read_tensor(p)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 5, 2)).astype("<f4")
    _blob(p, 4, x.shape, x.tobytes())
    np.testing.assert_array_equal(ingest.read_tensor(p), x)


def _ply(path, fields, rows, fmt="binary_little_endian", extra_elem=""):
    head = ["ply", f"format {fmt} 1.0", f"element vertex {len(rows)}"]
    head += [f"property {t} {n}" for n, t in fields]
    if extra_elem:
        head.append(extra_elem)
    head += ["end_header", ""]
    npt = {"float": "<f4", "double": "<f8", "uchar": "u1", "int": "<i4", "short": "<i2", "uint": "<u4"}
    rec = np.dtype([(n, npt[t]) for n, t in fields])
    body = np.array([tuple(r) for r in rows], dtype=rec)
    with open(path, "wb") as fh:
        fh.write("\n".join(head).encode())
        fh.write(body.tobytes())


def test_ply_variants_and_errors(tmp_path):
    p = tmp_path / "c.ply"
    rows = [(0.1, -2.0, 3.5, 7, 1, 2, 3), (1e-3, 4.25, -0.5, -9, 200, 100, 50)]
    _ply(p, [("x", "double"), ("y", "double"), ("z", "double"), ("label", "int"), ("red", "uchar"),
             ("green", "uchar"), ("blue", "uchar")], rows)
    pos, col = ingest.read_ply_points(p)
    np.testing.assert_array_equal(pos, np.array([r[:3] for r in rows], dtype=np.float64).astype(np.float32))
    np.testing.assert_array_equal(col, np.array([r[4:] for r in rows], dtype=np.uint8))
    _ply(p, [("z", "float"), ("y", "float"), ("x", "float")], [(1.0, 2.0, 3.0)])
    pos, col = ingest.read_ply_points(p)
    assert col is None and pos.tolist() == [[3.0, 2.0, 1.0]]
    with pytest.raises(BundleLoadError, match="missing point cloud"):
        ingest.read_ply_points(tmp_path / "none.ply")
    _ply(p, [("x", "float"), ("y", "float")], [(1.0, 2.0)])
    with pytest.raises(BundleStructureError, match="missing vertex property 'z'"):
        ingest.read_ply_points(p)
    _ply(p, [("x", "float"), ("y", "float"), ("z", "float")], [(1.0, 2.0, 3.0)], fmt="ascii")
    with pytest.raises(BundleStructureError, match="only binary_little_endian"):
        ingest.read_ply_points(p)
    _ply(p, [("x", "float"), ("y", "float"), ("z", "float")], [(1.0, 2.0, 3.0)], extra_elem="element face 3")
    with pytest.raises(BundleStructureError, match="unsupported PLY element 'face'"):
        ingest.read_ply_points(p)
    _ply(p, [("x", "float"), ("y", "float"), ("z", "float")], [(1.0, 2.0, 3.0)])
    p.write_bytes(p.read_bytes()[:-2])
    with pytest.raises(BundleStructureError, match="PLY body is 10 bytes, expected 12"):
        ingest.read_ply_points(p)
    p.write_bytes(b"not a ply")
    with pytest.raises(BundleStructureError, match="not a PLY file"):
        ingest.read_ply_points(p)
