"""Parity of the fused CUDA path (`fuse_and_query`) with the pinned CPU oracle.

Tolerances (BASELINE.json north_star):
* visibility bitset, visible counts, voxel codes: exact (mask pairs within 1e-6 of the depth-test
  threshold are exempt);
* fused features / similarities / softmax weights / properties / mass: 1e-4 relative in fp32
  (features per point as |a-b|/|b|; similarities as max_k|ds| <= 1e-4 * max(1e-2, max_k|s|)).
"""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from oracle import propfield_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-4
TOL_BF16 = 1e-2  # bf16-feature mode (tensor-core tile path: bf16 weights and G table)


def tol_for(wl, force_simt=False):
    """The tile path (bf16 maps, D % 128 == 0) computes in bf16 x bf16 -> fp32: 1e-2 bar."""
    return TOL_BF16 if (wl.cfg.bf16 and wl.cfg.d % 128 == 0 and not force_simt) else TOL


def run_gpu(wl, points=None, features=True, **kw):
    """features=True also writes the mean features, which bf16 maps compute with the feature-product
    tile kernel (k_tile_ws); features=False runs the production Gram kernel (pf_gram.cu)."""
    import torch

    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
    pts = wl.points if points is None else points
    res = pf.fuse_and_query(torch.from_numpy(np.ascontiguousarray(pts)).cuda(), views, tables,
                            temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid,
                            write_features=features, write_sims=True, write_weights=True, check=True, **kw)
    torch.cuda.synchronize()
    return res


def run_oracle(wl, points=None):
    pts = wl.points if points is None else points
    return O.fuse_and_query(pts, wl.views(f32_maps=True), wl.text, wl.values, wl.cfg.temperature,
                            wl.cfg.eps, wl.cfg.grid)


def knife_edge_pairs(wl, pts, eps):
    """(N, V) bool: pairs whose depth test sits within 1e-6 of its threshold."""
    p = np.asarray(pts, np.float64)
    out = np.zeros((p.shape[0], len(wl.poses)), dtype=bool)
    dep = wl.depth_np()
    for j, pose in enumerate(wl.poses):
        u, v, z = O.project_points(p, pose.rotation, pose.translation, wl.intrinsics.fx,
                                   wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy)
        h, w = dep[j].shape
        iu = np.clip(np.rint(u), 0, w - 1).astype(np.int64)
        iv = np.clip(np.rint(v), 0, h - 1).astype(np.int64)
        stored = dep[j][iv, iu].astype(np.float64)
        out[:, j] = np.abs(z - (stored + eps)) <= 1e-6
    return out


def assert_parity(res, ref, wl, pts=None, tol=TOL):
    pts = wl.points if pts is None else pts
    vis = res.visibility().cpu().numpy()
    diff = vis != ref["visibility"]
    if diff.any():
        assert not (diff & ~knife_edge_pairs(wl, pts, wl.cfg.eps)).any(), "mask mismatch"
    else:
        assert np.array_equal(res.counts.cpu().numpy(), ref["counts"])
    assert np.array_equal(res.codes.cpu().numpy(), ref["codes"])
    featured = ref["counts"] > 0
    if res.features is not None:  # features: per-point relative L2
        f = res.features.cpu().numpy().astype(np.float64)
        rf = ref["features"]
        rn = np.linalg.norm(rf, axis=1)
        rel = np.linalg.norm(f - rf, axis=1)[featured] / rn[featured]
        assert rel.max() <= tol, rel.max()
        assert np.all(f[~featured] == 0)
    s = res.sims.cpu().numpy().astype(np.float64)
    scale = np.maximum(1e-2, np.abs(ref["sims"]).max(axis=1))
    assert (np.abs(s - ref["sims"]).max(axis=1) <= tol * scale).all()
    w = res.weights.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(w, ref["weights"], rtol=tol, atol=tol * 1e-3)
    props = res.props.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(props, ref["props"], rtol=tol, atol=1e-6)
    assert res.mass_kg() == pytest.approx(ref["mass"], rel=tol)
    assert int(round(res.buffers.mass[1].item())) == ref["occupied"]
    part = res.host_partials()
    np.testing.assert_allclose(part["weight_totals"], ref["weights"].sum(axis=0), rtol=tol)
    pm = ref["weights"] @ wl.mid_theta
    assert part["pm_sum"] == pytest.approx(pm.sum(), rel=tol)
    np.testing.assert_allclose(part["pm_pos"], (pm[:, None] * pts.astype(np.float64)).sum(0), rtol=tol,
                               atol=tol * abs(pm.sum()))
    assert part["featured"] == int(featured.sum())
    assert part["visible_pairs"] == int(ref["counts"].sum())


@pytest.mark.parametrize("name", ["mini", "mini_bf16"])
def test_fused_vs_reference_goldens(cuda, golden, workload, name):
    """Against the reference's own outputs (golden fixtures), not just the oracle."""
    g = golden(name)
    wl = workload(name)
    for force, feats in ((False, True), (False, False), (True, True)):
        tol = tol_for(wl, force)
        res = run_gpu(wl, force_simt=force, features=feats)
        vis = np.unpackbits(g["visibility"], axis=1)[:, : wl.cfg.nviews].astype(bool)
        assert np.array_equal(res.visibility().cpu().numpy(), vis)
        assert np.array_equal(res.counts.cpu().numpy(), g["counts"])
        s = res.sims.cpu().numpy()
        scale = np.maximum(1e-2, np.abs(g["sims"]).max(axis=1))
        assert (np.abs(s - g["sims"]).max(axis=1) <= tol * scale).all()
        np.testing.assert_allclose(res.props.cpu().numpy(), g["props"], rtol=tol, atol=1e-6)


@pytest.mark.parametrize("features", [True, False])
@pytest.mark.parametrize("name", ["mini", "mini_bf16", "mini_fib40", "pr1"])
def test_fused_vs_oracle(cuda, workload, name, features):
    wl = workload(name)
    assert_parity(run_gpu(wl, features=features), run_oracle(wl), wl, tol=tol_for(wl))


def test_bf16_simt_path_meets_fp32_bar(cuda, workload):
    wl = workload("mini_bf16")
    assert_parity(run_gpu(wl, force_simt=True), run_oracle(wl), wl, tol=TOL)


@pytest.mark.parametrize("features", [True, False])
@pytest.mark.parametrize("name", ["c5", "c3"])
def test_tile_path_large_config_shapes(cuda, workload, name, features):
    """Tensor-core tile path on the real C5 / C3 view + map + material shapes (subset of points
    so the oracle finishes in seconds): masks / counts / codes exact, the rest at the bf16 bar.
    features=False: the Gram kernel; True: the feature-product kernel."""
    wl = workload(name, n=24_000)
    assert_parity(run_gpu(wl, features=features), run_oracle(wl), wl, tol=TOL_BF16)


def test_fused_c2_shapes_subset(cuda, workload):
    """C2 shapes (V=16 on two rings, 512^2, 37x37x768, K=32, 128^3) on 20k of its points."""
    wl = workload("c2", n=20_000)
    assert_parity(run_gpu(wl), run_oracle(wl), wl)


def test_tile_vs_simt_full_c5(cuda):
    """Full BASELINE C5 size (16M points x 64 views): the tile path's exact visibility (fp32 with
    error bound + fp64 fallback) must reproduce the fp64 SIMT path bit for bit; per-point
    properties and the voxel mass agree at the bf16 bar."""
    import torch

    from paper_2511_03126_b200 import workloads

    wl = workloads.generate("c5", device_splat=True)
    nv = wl.cfg.nviews
    R = np.stack([p.rotation for p in wl.poses])
    tv = np.stack([p.translation for p in wl.poses])
    intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
    fmap = torch.from_numpy(wl.fmaps.view(np.int16)).cuda().view(torch.bfloat16)
    views = pf.ViewSet.from_tensors(R, tv, intr, wl.depth.cuda(), fmap)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    pts = torch.from_numpy(wl.points).cuda()
    a = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid, check=True)
    ca, ma, pa, ka, mass_a = (a.counts.clone(), a.mask_bits.clone(), a.props.clone(), a.codes.clone(),
                              a.mass_kg())
    b = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid, force_simt=True, check=True)
    assert torch.equal(ca, b.counts)
    assert torch.equal(ma, b.mask_bits)
    assert torch.equal(ka, b.codes)
    feat = b.counts > 0
    rel = ((pa[:, 0] - b.props[:, 0]).abs() / b.props[:, 0].abs().clamp_min(1e-30))[feat]
    assert float(rel.max()) <= TOL_BF16
    assert mass_a == pytest.approx(b.mass_kg(), rel=TOL_BF16)


def test_tile_vs_simt_full_c3(cuda):
    """Full BASELINE C3 (2M points on 3 intersecting ellipsoids x 32 Fibonacci views, 1024^2 depth,
    74x74x1024 bf16 maps): tile path == fp64 SIMT path for bitsets / counts / codes, properties and
    mass at the bf16 bar."""
    import torch

    from paper_2511_03126_b200 import workloads

    wl = workloads.generate("c3", device_splat=True)
    nv = wl.cfg.nviews
    R = np.stack([p.rotation for p in wl.poses])
    tv = np.stack([p.translation for p in wl.poses])
    intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
    fmap = torch.from_numpy(wl.fmaps.view(np.int16)).cuda().view(torch.bfloat16)
    views = pf.ViewSet.from_tensors(R, tv, intr, wl.depth.cuda(), fmap)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    pts = torch.from_numpy(wl.points).cuda()
    a = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid, check=True)
    ca, ma, pa, ka, mass_a = (a.counts.clone(), a.mask_bits.clone(), a.props.clone(), a.codes.clone(),
                              a.mass_kg())
    b = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid, force_simt=True, check=True)
    assert torch.equal(ca, b.counts)
    assert torch.equal(ma, b.mask_bits)
    assert torch.equal(ka, b.codes)
    feat = b.counts > 0
    rel = ((pa[:, 0] - b.props[:, 0]).abs() / b.props[:, 0].abs().clamp_min(1e-30))[feat]
    assert float(rel.max()) <= TOL_BF16
    assert mass_a == pytest.approx(b.mass_kg(), rel=TOL_BF16)


def test_fused_c2_full_vs_oracle(cuda, workload):
    """Full BASELINE C2 object (200k points x 16 views, 37x37x768 f32, K=32, 128^3) against the CPU
    oracle at the fp32 bar (the SIMT path in Hilbert order)."""
    wl = workload("c2")
    assert_parity(run_gpu(wl), run_oracle(wl), wl)


@pytest.mark.parametrize("name", ["c4", "c2"])
def test_x3_tile_path_full_object(cuda, workload, name):
    """f32 maps at full object size take the tensor-core tile path in x3 mode (bf16 hi/lo operand
    splits, three MMAs per k-step): the fp32 bar against the oracle, and masks / counts / codes
    identical to the fp64 SIMT path."""
    import torch

    wl = workload(name)
    res = run_gpu(wl)
    assert_parity(res, run_oracle(wl), wl)
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
    pts = torch.from_numpy(wl.points).cuda()
    a = pf.fuse_and_query(pts, views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid)
    ca, ma, pa = a.counts.clone(), a.mask_bits.clone(), a.props.clone()
    b = pf.fuse_and_query(pts, views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid,
                          force_simt=True)
    assert torch.equal(ca, b.counts) and torch.equal(ma, b.mask_bits)
    feat = b.counts > 0
    rel = ((pa[:, 0] - b.props[:, 0]).abs() / b.props[:, 0].abs().clamp_min(1e-30))[feat]
    assert float(rel.max()) <= TOL


def test_featureless_points(cuda, workload):
    """Points seen by no view: zero probability/property rows, still voxel-occupying (rho=0)."""
    wl = workload("mini")
    far = np.array([[0.0, 0.0, 50.0], [40.0, 0.0, 0.0], [0.0, -60.0, 1.0]], dtype=np.float32)
    pts = np.concatenate([wl.points, far])
    res = run_gpu(wl, points=pts)
    ref = run_oracle(wl, points=pts)
    assert (ref["counts"][-3:] == 0).all()
    assert_parity(res, ref, wl, pts)
    assert np.all(res.props.cpu().numpy()[-3:] == 0)
    assert np.all(res.weights.cpu().numpy()[-3:] == 0)


def test_empty_point_set(cuda, workload):
    import torch

    wl = workload("mini")
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    res = pf.fuse_and_query(torch.zeros((0, 3), device="cuda"), views, tables, grid=8)
    assert res.props.shape[0] == 0 and res.mass_kg() == 0.0


def test_single_point(cuda, workload):
    wl = workload("mini")
    pts = wl.points[:1].copy()
    assert_parity(run_gpu(wl, points=pts), run_oracle(wl, points=pts), wl, pts)


def test_permutation_equivariance_c2(cuda, workload):
    """Size-independent property at full C2 size: permuting points permutes per-point outputs
    and leaves the mass unchanged."""
    import torch

    wl = workload("c2")
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    pts = torch.from_numpy(wl.points).cuda()
    a = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid)
    pa, ma, ca = a.props.clone(), a.mass_kg(), a.counts.clone()
    perm = torch.randperm(pts.shape[0], device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    b = pf.fuse_and_query(pts[perm].contiguous(), views, tables, grid=wl.cfg.grid)
    assert torch.equal(b.counts, ca[perm])
    assert torch.allclose(b.props, pa[perm], rtol=1e-6, atol=1e-4)
    assert b.mass_kg() == pytest.approx(ma, rel=1e-5)
    # probabilities are a convex combination -> properties inside the material hull
    dens = b.props[:, 0][b.counts > 0]
    assert float(dens.min()) >= wl.density.min() - 1e-2 and float(dens.max()) <= wl.density.max() + 1e-2


def test_nan_similarity_raises(cuda, workload):
    import torch

    wl = workload("mini")
    views = wl.views()
    views[0].feature_map = np.full_like(views[0].feature_map, np.nan)
    vs = pf.ViewSet.from_views(views)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    with pytest.raises(pf.MaterialError):
        pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), vs, tables, grid=8, check=True)


@pytest.mark.parametrize("name", ["mini_bf16", "pr1"])
def test_sparse_voxel_mass_equals_dense_and_cleans_grid(workload, name):
    """The touched-voxel-list reduction (one GPU) equals the dense grid scan and leaves the grid
    zeroed, so buffers reused across objects need no memset."""
    import torch

    from paper_2511_03126_b200 import _lib
    from paper_2511_03126_b200.device import ptr, stream_handle

    wl = workload(name)
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
    pts = torch.from_numpy(np.ascontiguousarray(wl.points)).cuda()
    bufs = pf.FuseBuffers(pts.shape[0], views, tables, wl.cfg.grid)
    masses = []
    for _ in range(3):
        res = pf.fuse_and_query(pts, views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps,
                                grid=wl.cfg.grid, buffers=bufs, reduce=False)
        dense_grid = bufs.grid_partials.clone()
        dense = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.call("pf_voxel_mass", ptr(dense_grid), wl.cfg.grid, ptr(bufs.lo_hi), ptr(dense), stream_handle())
        res.finalize()
        torch.cuda.synchronize()
        assert abs(res.mass_kg() - dense[0].item()) <= 1e-12 * dense[0].item()
        assert int(round(bufs.mass[1].item())) == int(round(dense[1].item()))
        assert not bool(bufs.grid_partials.any())
        masses.append(res.mass_kg())
    assert max(masses) - min(masses) <= 1e-6 * masses[0]  # fp32 atomics: order-dependent rounding


@pytest.mark.parametrize("n", [1, 127, 129, 511, 513, 1025])
def test_gram_tile_boundaries(cuda, workload, n):
    """Point counts around the 128-row and 512-row tile edges on the Gram path (a short last 512-row
    tile must stay a Gram item; its 128-row tiles and 32-row splits must cover every row once)."""
    wl = workload("mini_bf16")
    assert wl.points.shape[0] >= n
    pts = np.ascontiguousarray(wl.points[:n])
    assert_parity(run_gpu(wl, pts, features=False), run_oracle(wl, pts), wl, pts, tol=TOL_BF16)


@pytest.mark.parametrize("name,features", [("mini_bf16", False), ("mini_bf16", True), ("mini", True)])
def test_views_with_different_depth_sizes(cuda, workload, name, features):
    """Depth maps of different sizes per view (the feature maps stay uniform, as the tile path needs):
    odd views get their depth zero-padded to a larger W x H, which changes their feature-coordinate
    scale Wf / W (fusion.py:83-86) and adds never-visible pixels. Gram, feature-product and SIMT
    paths against the oracle on the same view list."""
    import dataclasses

    import torch

    wl = workload(name)
    vg, vo = wl.views(), wl.views(f32_maps=True)
    for j in range(1, len(vg), 2):
        dep = np.pad(vg[j].depth, ((0, 13), (0, 7)))
        vg[j] = dataclasses.replace(vg[j], depth=dep)
        vo[j] = dataclasses.replace(vo[j], depth=dep)
    views = pf.ViewSet.from_views(vg)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=wl.cfg.temperature,
                            epsilon=wl.cfg.eps, grid=wl.cfg.grid, write_features=features, write_sims=True,
                            write_weights=True, check=True)
    torch.cuda.synchronize()
    ref = O.fuse_and_query(wl.points, vo, wl.text, wl.values, wl.cfg.temperature, wl.cfg.eps, wl.cfg.grid)
    assert np.array_equal(res.counts.cpu().numpy(), ref["counts"])
    assert np.array_equal(res.codes.cpu().numpy(), ref["codes"])
    tol = tol_for(wl)
    props = res.props.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(props, ref["props"], rtol=tol, atol=1e-6)
    assert res.mass_kg() == pytest.approx(ref["mass"], rel=tol)


@pytest.mark.parametrize("name", ["mini_bf16", "mini"])
def test_camera_inside_the_point_cloud(cuda, workload, name):
    """One view's camera sits at the centre of the object, so points lie in front of, beside and
    behind its image plane (tiles that reach z <= 0 take the exact per-point test; the depth map is
    the reference's own visibility rule applied to whatever it stores). Tile / SIMT paths against the
    oracle on the same views."""
    import dataclasses

    import torch

    from paper_2511_03126_b200.types import CameraPose

    wl = workload(name)
    vg, vo = wl.views(), wl.views(f32_maps=True)
    c = wl.points.astype(np.float64).mean(axis=0)
    rot = np.asarray(vg[0].camera.rotation)
    cam = CameraPose(rotation=rot, translation=-rot @ c)
    dep = np.full_like(vg[0].depth, 0.05)  # a near wall: only points within 0.05 + eps in front pass
    vg[0] = dataclasses.replace(vg[0], camera=cam, depth=dep)
    vo[0] = dataclasses.replace(vo[0], camera=cam, depth=dep)
    views = pf.ViewSet.from_views(vg)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=wl.cfg.temperature,
                            epsilon=wl.cfg.eps, grid=wl.cfg.grid, check=True)
    torch.cuda.synchronize()
    ref = O.fuse_and_query(wl.points, vo, wl.text, wl.values, wl.cfg.temperature, wl.cfg.eps, wl.cfg.grid)
    assert np.array_equal(res.visibility().cpu().numpy(), ref["visibility"])
    assert np.array_equal(res.counts.cpu().numpy(), ref["counts"])
    assert np.array_equal(res.codes.cpu().numpy(), ref["codes"])
    tol = tol_for(wl)
    np.testing.assert_allclose(res.props.cpu().numpy().astype(np.float64), ref["props"], rtol=tol, atol=1e-6)
