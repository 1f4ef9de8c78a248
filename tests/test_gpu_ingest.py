"""load_bundle_device: a bundle written by the reference's save_bundle lands in the
packed device layout exactly as the reference's load_bundle values (tests/golden/bundle_tiny.npz),
and the fused path on it equals the path on views packed from those arrays."""

import os
import shutil

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from paper_2511_03126_b200 import ingest
from paper_2511_03126_b200.errors import BundleLoadError, BundleStructureError
from paper_2511_03126_b200.types import CameraPose, Intrinsics, ViewRecord

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
BUNDLE = os.path.join(HERE, "golden", "bundle_tiny")


def test_load_bundle_device_matches_reference(cuda, golden):
    import torch

    g = golden("bundle_tiny")
    b = ingest.load_bundle_device(BUNDLE)
    v = b.views
    assert v.nviews == 3 and v.d == 32 and b.scene_id == "tiny" and b.gt_mass_kg == 1.25
    torch.testing.assert_close(v.depth.cpu(), torch.from_numpy(g["depth"].reshape(-1)), rtol=0, atol=0)
    torch.testing.assert_close(v.fmap.cpu(), torch.from_numpy(g["features"].reshape(-1)), rtol=0, atol=0)
    np.testing.assert_array_equal(b.points.cpu().numpy(), g["positions"])
    np.testing.assert_array_equal(b.colors, g["colors"])
    np.testing.assert_array_equal(v.records["R"].reshape(3, 3, 3), g["rotations"])
    np.testing.assert_array_equal(v.records["t"], g["translations"])
    assert [e.name for e in b.material_dictionary.entries] == ["wood", "steel"]
    assert b.material_dictionary.entries[0].properties["density"] == (500.0, 700.0)
    assert len(b.reference_poses) == 3
    # the fused path on the loaded bundle == on views packed from the reference's arrays
    views = [ViewRecord(depth=g["depth"][j], camera=CameraPose(rotation=g["rotations"][j], translation=g["translations"][j]),
                        intrinsics=Intrinsics(*g["intrinsics"][j]), feature_map=g["features"][j]) for j in range(3)]
    ref_views = pf.ViewSet.from_views(views)
    rng = np.random.default_rng(0)
    text = rng.standard_normal((4, 32)).astype(np.float32)
    text /= np.linalg.norm(text, axis=1, keepdims=True)
    tables = pf.QueryTables.build(text, rng.uniform(100, 8000, (4, 2)).astype(np.float32))
    a = pf.fuse_and_query(b.points, v, tables, grid=16)
    r = pf.fuse_and_query(torch.from_numpy(g["positions"]).cuda(), ref_views, tables, grid=16)
    assert torch.equal(a.counts, r.counts) and torch.equal(a.mask_bits, r.mask_bits)
    assert torch.equal(a.props, r.props)
    # voxel sums are fp32 atomics: the accumulation order (and so the last bits) varies run to run
    assert a.mass_kg() == pytest.approx(r.mass_kg(), rel=1e-6)
    b2 = ingest.load_bundle_device(BUNDLE, view_limit=2, fmap_kind="bf16")
    assert b2.views.nviews == 2 and b2.views.fmap.dtype == torch.bfloat16 and len(b2.reference_poses) == 2


def test_load_bundle_device_errors(cuda, tmp_path):
    with pytest.raises(BundleLoadError, match="missing manifest"):
        ingest.load_bundle_device(tmp_path)
    d = tmp_path / "b"
    shutil.copytree(BUNDLE, d)
    os.remove(d / "views" / "1" / "feat.f32")
    with pytest.raises(BundleLoadError, match="missing tensor blob"):
        ingest.load_bundle_device(d)
    shutil.copy(d / "views" / "0" / "depth.f32", d / "views" / "1" / "feat.f32")
    with pytest.raises(BundleStructureError, match="feature blob for view 1 has rank 2"):
        ingest.load_bundle_device(d)
    os.remove(d / "views" / "2" / "image.png")
    shutil.copy(d / "views" / "0" / "feat.f32", d / "views" / "1" / "feat.f32")
    with pytest.raises(BundleLoadError, match="missing image"):
        ingest.load_bundle_device(d)
