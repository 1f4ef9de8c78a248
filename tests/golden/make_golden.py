"""Generate golden vectors by running the REFERENCE implementation (propfield, read-only mount).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified reference, feeds it seeded inputs (tests/golden/recipes.py and the
`mini` / `mini_bf16` workloads of paper_2511_03126_b200.workloads), and writes its outputs as
small .npz fixtures next to this file. The tests compare both the CPU oracle (oracle/) and the
CUDA path against these files; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")

import recipes  # noqa: E402
from paper_2511_03126_b200 import workloads  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_views(wl, propfield):
    from propfield.bundle import CameraPose, Intrinsics, ViewRecord

    dep = wl.depth_np()
    fm = wl.fmaps_f32()
    out = []
    for j, pose in enumerate(wl.poses):
        h, w = dep[j].shape
        out.append(
            ViewRecord(
                image=np.zeros((h, w, 3), dtype=np.uint8),
                depth=dep[j],
                camera=CameraPose(rotation=pose.rotation, translation=pose.translation),
                intrinsics=Intrinsics(fx=wl.intrinsics.fx, fy=wl.intrinsics.fy,
                                      cx=wl.intrinsics.cx, cy=wl.intrinsics.cy),
                feature_map=fm[j],
            )
        )
    return out


def kernels_golden(numpy_impl):
    u, v, z, depth = recipes.visible_case()
    vis0 = numpy_impl.visible_in_view(u, v, z, depth, 0.0)
    vis5 = numpy_impl.visible_in_view(u, v, z, depth, 0.05)
    fmap, fu, fv = recipes.gather_case()
    gath = numpy_impl.bilinear_gather(fmap, fu, fv)
    fmap2, fu2, fv2, rows = recipes.accumulate_case()
    acc = np.zeros((300, 4))
    cnt = np.zeros(300, dtype=np.int64)
    numpy_impl.accumulate_features(fmap2, fu2, fv2, rows, acc, cnt)
    return dict(visible_eps0=np.packbits(vis0), visible_eps005=np.packbits(vis5),
                gather=gath, accum=acc, accum_counts=cnt)


def grounding_golden(grounding):
    out = {}
    for seed in range(2):
        f, t, y = recipes.grounding_case(seed)
        s = grounding.material_similarity(f, t)
        w = grounding.softmax_weights(s, 0.1)
        out[f"sims{seed}"] = s
        out[f"weights{seed}"] = w
        out[f"props{seed}"] = grounding.regress_with_weights(w, y)
        out[f"kreg{seed}"] = grounding.kernel_regress(s, y[:, 0], 0.05)
    return out


def pipeline_golden(name, propfield):
    from propfield import fusion, geometry, grounding, integrate
    from propfield.densify import PropertyField
    from propfield.grounding import MaterialDictionary, MaterialEntry

    wl = workloads.generate(name)
    cfg = wl.cfg
    views = ref_views(wl, propfield)
    pos = wl.points.astype(np.float64)
    vis = geometry.visibility_mask(pos, views, cfg.eps)
    sem = fusion.aggregate_geometric_features(pos, views, vis)
    feats = sem.features
    norm = np.linalg.norm(feats, axis=1, keepdims=True)
    fhat = np.where(norm > 0, feats / np.where(norm > 0, norm, 1.0), 0.0)  # fusion.py:210-214
    featured = sem.visible_counts > 0
    text = wl.text.astype(np.float64)
    sims = np.zeros((len(pos), cfg.k))
    weights = np.zeros((len(pos), cfg.k))
    sims[featured] = grounding.material_similarity(fhat[featured], text)
    weights[featured] = grounding.softmax_weights(sims[featured], cfg.temperature)
    props = grounding.regress_with_weights(weights, wl.values)
    # integrate_mass on the same probabilities (integrate.py:98-167)
    entries = [
        MaterialEntry(name=f"m{k}", properties={"density": (float(wl.density[k]), float(wl.density[k]))},
                      thickness_m=float(wl.thickness[k]))
        for k in range(cfg.k)
    ]
    fld = PropertyField(positions=wl.points, probabilities=weights,
                        dominant=weights.argmax(axis=1), properties={}, material_names=[e.name for e in entries])
    est = integrate.integrate_mass(fld, MaterialDictionary(entries=entries), integrate.IntegrationConfig())
    out = dict(
        visibility=np.packbits(vis, axis=1), counts=sem.visible_counts, sims=sims, weights=weights,
        props=props, feature_norms=norm[:, 0], features_sha=np.array(sha(feats)),
        integ_mass=np.array(est.mass_kg), integ_length=np.array(est.characteristic_length),
        integ_b=np.array(est.b_adap), integ_com=np.asarray(est.center_of_mass),
        integ_per_material=np.array([est.per_material[e.name] for e in entries]),
    )
    if feats.nbytes <= 1_100_000:
        out["features"] = feats
    else:
        rows = np.random.default_rng(7).choice(len(pos), 64, replace=False)
        out["feature_rows"] = rows
        out["features_subset"] = feats[rows]
    return out


def densify_golden():
    """dino_knn_interpolate on recipes.densify_cases() and densify_field on densify_field_case()."""
    from propfield.densify import densify_field, dino_knn_interpolate
    from propfield.fusion import SemanticPointCloud
    from propfield.grounding import MaterialDictionary, MaterialEntry
    from propfield.sampling import SourcePointSet

    out = {}
    for name, q, s, p, k in recipes.densify_cases():
        out[f"dk_{name}"] = dino_knn_interpolate(q, s, p, k)
    c = recipes.densify_field_case()
    n = c["positions"].shape[0]
    semantic = SemanticPointCloud(positions=c["positions"], features=c["features"], visible_counts=c["counts"],
                                  visibility=(c["counts"] > 0)[:, None])
    src = SourcePointSet(indices=c["src_pick"], positions=c["positions"][c["src_pick"]], voxel_size=0.1,
                         features=c["src_features"], probabilities=c["src_probs"])
    entries = [MaterialEntry(name=nm, properties={"density": tuple(c["density"][i]), "hardness": tuple(c["hardness"][i])},
                             thickness_m=0.01) for i, nm in enumerate(["wood", "steel"])]
    fld = densify_field(semantic, src, MaterialDictionary(entries=entries), k=3)
    out["df_probabilities"] = fld.probabilities
    out["df_dominant"] = fld.dominant
    out["df_density"] = fld.properties["density"]
    out["df_hardness"] = fld.properties["hardness"]
    out["df_featureless"] = fld.flags["featureless"]
    assert n == len(fld)
    return out


def bundle_golden(out_dir):
    """A tiny capture bundle written by the reference's own save_bundle (bundle.py:262-305): 3 views
    of 48x48 depth / 6x6x32 features, 300 points with colours, materials and reference poses."""
    import shutil

    from propfield.bundle import CameraPose, CaptureBundle, Intrinsics, PointCloud, ViewRecord, save_bundle
    from propfield.grounding import MaterialDictionary, MaterialEntry

    rng = np.random.default_rng(21)
    pts = workloads.sample_ellipsoid(rng, 300, (0.3, 0.25, 0.2)).astype(np.float32)
    intr = Intrinsics(fx=48.0, fy=48.0, cx=24.0, cy=24.0)
    views, ref = [], []
    for j, az in enumerate((0.0, 2.1, 4.2)):
        eye = np.array([1.5 * np.cos(az), 1.5 * np.sin(az), 0.5])
        pose = workloads.look_at_pose(np.zeros(3), eye)
        cam = CameraPose(rotation=pose.rotation, translation=pose.translation)
        ref.append(cam)
        depth = workloads.splat_depth(pts.astype(np.float64), pose, intr, 48, 48)
        feat = rng.standard_normal((6, 6, 32)).astype(np.float32)
        img = rng.integers(0, 255, (48, 48, 3), dtype=np.uint8)
        views.append(ViewRecord(image=img, depth=depth, camera=cam, intrinsics=intr, feature_map=feat))
    cloud = PointCloud(positions=pts, colors=rng.integers(0, 255, (300, 3), dtype=np.uint8))
    mats = MaterialDictionary(entries=[
        MaterialEntry(name="wood", properties={"density": (500.0, 700.0), "hardness": (0.3, 0.3)}, thickness_m=0.02),
        MaterialEntry(name="steel", properties={"density": (7800.0, 7800.0), "hardness": (0.9, 0.95)},
                      thickness_m=0.002)])
    bundle = CaptureBundle(views=views, point_cloud=cloud, reference_poses=ref, material_dictionary=mats,
                           scene_id="tiny", gt_mass_kg=1.25)
    if os.path.isdir(out_dir):
        shutil.rmtree(out_dir)
    save_bundle(bundle, out_dir)
    # what the reference's load_bundle returns for it (pins the native readers in tests/test_ingest.py)
    from propfield.bundle import load_bundle

    back = load_bundle(out_dir)
    np.savez_compressed(out_dir + ".npz", depth=np.stack([v.depth for v in back.views]),
                        features=np.stack([v.feature_map for v in back.views]),
                        positions=back.point_cloud.positions, colors=back.point_cloud.colors,
                        rotations=np.stack([v.camera.rotation for v in back.views]),
                        translations=np.stack([v.camera.translation for v in back.views]),
                        intrinsics=np.array([[v.intrinsics.fx, v.intrinsics.fy, v.intrinsics.cx, v.intrinsics.cy]
                                             for v in back.views]))


def normals_golden():
    from propfield.geometry import estimate_normals

    out = {}
    for name, p, cams, k in recipes.normals_cases():
        nrm, deg = estimate_normals(p, k, cams)
        out[f"n_{name}"] = nrm
        out[f"d_{name}"] = deg
    return out


def views_golden(propfield):
    """score_views / rank_views (view_select.py:51-124) on 150 anchors of the `mini` workload."""
    from propfield import geometry
    from propfield.sampling import SourcePointSet
    from propfield.view_select import rank_views, score_views

    wl = workloads.generate("mini")
    views = ref_views(wl, propfield)
    pos = wl.points.astype(np.float64)
    centers = np.stack([v.camera.center for v in views])
    normals, _ = geometry.estimate_normals(pos, 16, centers)
    idx = np.random.default_rng(5).choice(len(pos), 150, replace=False)
    vis = geometry.visibility_mask(pos[idx], views, wl.cfg.eps)
    vis[:3] = False  # anchors visible nowhere
    src = SourcePointSet(indices=idx, positions=pos[idx], voxel_size=0.1, normals=normals[idx])
    st, sa, z, px = score_views(src, views, vis)
    ranks = rank_views(src, views, vis, 3)
    ranked = np.full((150, 3), -1, np.int32)
    for i, r in enumerate(ranks):
        for q, e in enumerate(r):
            ranked[i, q] = e.view_index
    return dict(indices=idx, normals=normals[idx], visibility=vis, s_total=st, s_angle=sa, z=z, pixels=px,
                ranked=ranked, zero_visible=src.flags["zero_visible"])


def main():
    import propfield  # noqa: F401  (the unmodified reference)
    from propfield import grounding
    from propfield.kernels import numpy_impl

    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernels_golden(numpy_impl))
    np.savez_compressed(os.path.join(HERE, "grounding.npz"), **grounding_golden(grounding))
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **densify_golden())
    bundle_golden(os.path.join(HERE, "bundle_tiny"))
    np.savez_compressed(os.path.join(HERE, "normals.npz"), **normals_golden())
    np.savez_compressed(os.path.join(HERE, "views.npz"), **views_golden(propfield))
    for name in ("mini", "mini_bf16"):
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **pipeline_golden(name, propfield))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
