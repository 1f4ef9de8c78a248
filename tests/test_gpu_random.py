"""Randomised shape sweep of the fused path against the CPU oracle (seeded): point counts from 1 to
~70k, 1..64 views (rings or Fibonacci spheres, clutter of 1-3 ellipsoids), image and feature-grid
sizes, D in {64, 128, 256, 384}, K in 1..128, P in 1..4 properties, temperatures 0.05..1, grid sides
1..48, f32 and bf16 maps — which exercises the SIMT path, the bf16 tile path and (from 64k points
with f32 maps and D % 128 == 0) the x3 tile path. Bars as in test_gpu_fused: masks / counts / codes
exact (knife-edge pairs exempt), properties 1e-4 (f32) / 1e-2 (bf16 tile path), voxel mass."""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from oracle import propfield_oracle as O
from paper_2511_03126_b200 import workloads
from test_gpu_fused import knife_edge_pairs

pytestmark = pytest.mark.gpu


def _config(seed):
    rng = np.random.default_rng(1000 + seed)
    views = int(rng.choice([1, 2, 5, 8, 17, 32, 64]))
    use_rings = bool(rng.integers(0, 2)) and views >= 2
    d = int(rng.choice([64, 128, 256, 384]))
    hf = int(rng.integers(3, 20))
    wf = int(rng.integers(3, 20))
    n = int(rng.choice([1, 7, 300, 2000, 9000]))
    if seed == 11:  # the x3 path (f32, >= 64k points, D % 128 == 0)
        n, d, views, use_rings = 70_000, 128, 6, False
    bf16 = bool(rng.integers(0, 2)) and seed != 11
    cfg = workloads.Config(
        f"rand{seed}", n=n, rings=((views // 2, 15.0), (views - views // 2, 45.0)) if use_rings else (),
        fib=0 if use_rings else views, radius=float(rng.uniform(1.2, 2.5)), image=int(rng.choice([48, 64, 96, 128])),
        fmap=(hf, wf, d), bf16=bf16, k=int(rng.integers(1, 129)), grid=int(rng.integers(1, 49)),
        n_ellipsoids=int(rng.integers(1, 4)), temperature=float(rng.uniform(0.05, 1.0)), seed=seed)
    p = int(rng.integers(1, 5))
    return cfg, p, rng


@pytest.mark.parametrize("seed", range(128))
def test_random_shapes_vs_oracle(cuda, seed):
    import torch

    cfg, p, rng = _config(seed)
    wl = workloads.generate(cfg)
    values = np.column_stack([wl.density] + [rng.uniform(0, 1, cfg.k) for _ in range(p - 1)])
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, values.astype(np.float32), wl.mid_theta)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=cfg.temperature,
                            epsilon=cfg.eps, grid=cfg.grid, check=True)
    ref = O.fuse_and_query(wl.points, wl.views(f32_maps=True), wl.text, values, cfg.temperature, cfg.eps, cfg.grid)
    vis = res.visibility().cpu().numpy()
    diff = vis != ref["visibility"]
    if diff.any():
        assert not (diff & ~knife_edge_pairs(wl, wl.points, cfg.eps)).any(), "mask mismatch"
    np.testing.assert_array_equal(res.codes.cpu().numpy(), ref["codes"])
    cnt = res.counts.cpu().numpy()
    if not diff.any():
        np.testing.assert_array_equal(cnt, ref["counts"])
    tile_bf16 = cfg.bf16 and cfg.d % 128 == 0 and cfg.nviews <= 64 and cfg.k <= 128
    tol = 1e-2 if tile_bf16 else 1e-4
    props = res.props.cpu().numpy().astype(np.float64)
    scale = np.abs(ref["props"]).max(axis=0, keepdims=True) + 1e-30
    assert (np.abs(props - ref["props"]) / scale).max() <= tol, (cfg, p)
    assert res.mass_kg() == pytest.approx(ref["mass"], rel=tol, abs=1e-12)


@pytest.mark.parametrize("seed", range(32))
def test_random_medium_bf16_gram_vs_oracle(cuda, seed):
    """Medium objects (100k-250k points, bf16 maps, D % 128 == 0) through the production Gram path:
    several 512-row tiles per object, 128 / 32-row splits and SIMT overflow in one call, against
    the oracle run on every host core (tests/oracle_parallel.py)."""
    import torch

    from oracle_parallel import oracle_rows, unpack_mask_bits

    rng = np.random.default_rng(5000 + seed)
    views = int(rng.choice([8, 17, 32, 64]))
    cfg = workloads.Config(
        f"medium{seed}", n=int(rng.choice([100_000, 250_000])), rings=(), fib=views,
        radius=float(rng.uniform(1.2, 2.5)), image=int(rng.choice([128, 256])),
        fmap=(int(rng.integers(8, 40)), int(rng.integers(8, 40)), int(rng.choice([128, 256, 512]))), bf16=True,
        k=int(rng.integers(1, 129)), grid=int(rng.integers(8, 128)), n_ellipsoids=int(rng.integers(1, 4)),
        temperature=float(rng.uniform(0.05, 1.0)), seed=seed)
    wl = workloads.generate(cfg)
    views_dev = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views_dev, tables, temperature=cfg.temperature,
                            epsilon=cfg.eps, grid=cfg.grid, check=True)
    torch.cuda.synchronize()
    ref = oracle_rows(wl)
    vis_g = unpack_mask_bits(res.mask_bits.cpu().numpy(), cfg.nviews)
    vis_r = np.unpackbits(ref["vis_bits"], axis=1, bitorder="little")[:, :cfg.nviews].astype(bool)
    diff = vis_g != vis_r
    if diff.any():
        assert not (diff & ~knife_edge_pairs(wl, wl.points, cfg.eps)).any(), "mask mismatch"
    np.testing.assert_array_equal(res.codes.cpu().numpy(), ref["codes"])
    ok = ~diff.any(axis=1)
    np.testing.assert_array_equal(res.counts.cpu().numpy()[ok], ref["counts"][ok])
    props = res.props.cpu().numpy().astype(np.float64)
    scale = np.abs(ref["props"]).max(axis=0, keepdims=True) + 1e-30
    assert (np.abs(props - ref["props"])[ok] / scale).max() <= 1e-2, cfg
    np.testing.assert_allclose(res.host_partials()["weight_totals"], ref["weight_totals"], rtol=1e-2)


@pytest.mark.parametrize("seed", range(12))
def test_random_medium_f32_x3_vs_oracle(cuda, seed):
    """Medium objects with f32 maps (70k-150k points, D % 128 == 0): the x3 tile path (hi / lo bf16
    splits in the feature-product kernel) against the parallel oracle at the fp32 bar."""
    import torch

    from oracle_parallel import oracle_rows, unpack_mask_bits

    rng = np.random.default_rng(7000 + seed)
    views = int(rng.choice([4, 8, 17, 32]))
    cfg = workloads.Config(
        f"medium_f32_{seed}", n=int(rng.choice([70_000, 150_000])), rings=(), fib=views,
        radius=float(rng.uniform(1.2, 2.5)), image=int(rng.choice([96, 128, 192])),
        fmap=(int(rng.integers(8, 24)), int(rng.integers(8, 24)), int(rng.choice([128, 256]))), bf16=False,
        k=int(rng.integers(1, 129)), grid=int(rng.integers(8, 96)), n_ellipsoids=int(rng.integers(1, 4)),
        temperature=float(rng.uniform(0.05, 1.0)), seed=seed)
    wl = workloads.generate(cfg)
    views_dev = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views_dev, tables, temperature=cfg.temperature,
                            epsilon=cfg.eps, grid=cfg.grid, check=True)
    torch.cuda.synchronize()
    ref = oracle_rows(wl)
    vis_g = unpack_mask_bits(res.mask_bits.cpu().numpy(), cfg.nviews)
    vis_r = np.unpackbits(ref["vis_bits"], axis=1, bitorder="little")[:, :cfg.nviews].astype(bool)
    diff = vis_g != vis_r
    if diff.any():
        assert not (diff & ~knife_edge_pairs(wl, wl.points, cfg.eps)).any(), "mask mismatch"
    np.testing.assert_array_equal(res.codes.cpu().numpy(), ref["codes"])
    ok = ~diff.any(axis=1)
    np.testing.assert_array_equal(res.counts.cpu().numpy()[ok], ref["counts"][ok])
    props = res.props.cpu().numpy().astype(np.float64)
    scale = np.abs(ref["props"]).max(axis=0, keepdims=True) + 1e-30
    assert (np.abs(props - ref["props"])[ok] / scale).max() <= 1e-4, cfg
    np.testing.assert_allclose(res.host_partials()["weight_totals"], ref["weight_totals"], rtol=1e-4)
