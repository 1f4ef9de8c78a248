"""Full-size objects of the bf16 configs against the CPU oracle.

The GPU runs the whole object through the production path (Gram tile kernel, 512-point tiles,
128 / 32-row splits, SIMT overflow), so the tile regime is the one the benchmark measures. The
oracle (reference algorithm, numpy/numba fp64; tests/oracle_parallel.py splits the points over the
host's cores) runs on:
* C3 (2M points x 32 views, 74x74x1024 bf16): every point, mass included;
* C5 (16M points x 64 views, 37x37x1024 bf16): a stratified slice of every 8th sorted-by-index
  point (2M points), voxel codes over the full object's domain; the C5 mass is checked against
  the fp64-visibility SIMT kernel on the same object (test_gpu_fused::test_tile_vs_simt_full_c5).
Bars (BASELINE north_star, bf16-feature mode): visibility bit-exact except pairs within 1e-6 of the
depth threshold, counts and voxel codes exact, properties and mass 1e-2 relative.

The SIMT kernel's D = 1024 bf16 instantiation (k_fuse_simt<1, 8, 4>, used for overflow tiles) is
checked on its own at the fp32 bar on a C5-shaped subset.
"""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from oracle import propfield_oracle as O
from oracle_parallel import oracle_rows, unpack_mask_bits

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2


def _gpu_full(wl):
    import torch

    nv = wl.cfg.nviews
    R = np.stack([p.rotation for p in wl.poses])
    tv = np.stack([p.translation for p in wl.poses])
    intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
    fmap = torch.from_numpy(wl.fmaps.view(np.int16)).cuda().view(torch.bfloat16)
    depth = wl.depth if hasattr(wl.depth, "cuda") else torch.from_numpy(wl.depth)
    views = pf.ViewSet.from_tensors(R, tv, intr, depth.cuda(), fmap)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=wl.cfg.temperature,
                            epsilon=wl.cfg.eps, grid=wl.cfg.grid, check=True)
    torch.cuda.synchronize()
    return {"mask": res.mask_bits.cpu().numpy(), "counts": res.counts.cpu().numpy(),
            "props": res.props.cpu().numpy().astype(np.float64), "codes": res.codes.cpu().numpy(),
            "mass": res.mass_kg(), "partials": res.host_partials()}


def _knife_edge(wl, idx, rows_cols):
    """For (row, view) pairs: is |z - (stored + eps)| <= 1e-6 (fp64, the reference arithmetic)?"""
    dep = wl.depth_np()
    out = np.zeros(len(rows_cols), dtype=bool)
    for j in np.unique(rows_cols[:, 1]):
        sel = rows_cols[:, 1] == j
        p = wl.points[idx[rows_cols[sel, 0]]].astype(np.float64)
        pose = wl.poses[j]
        u, v, z = O.project_points(p, pose.rotation, pose.translation, wl.intrinsics.fx, wl.intrinsics.fy,
                                   wl.intrinsics.cx, wl.intrinsics.cy)
        h, w = dep[j].shape
        iu = np.clip(np.rint(u), 0, w - 1).astype(np.int64)
        iv = np.clip(np.rint(v), 0, h - 1).astype(np.int64)
        out[sel] = np.abs(z - (dep[j][iv, iu].astype(np.float64) + wl.cfg.eps)) <= 1e-6
    return out


def _check_rows(wl, g, ref):
    idx = ref["idx"]
    nv = wl.cfg.nviews
    vis_g = unpack_mask_bits(g["mask"][idx], nv)
    vis_r = np.unpackbits(ref["vis_bits"], axis=1, bitorder="little")[:, :nv].astype(bool)
    diff = np.argwhere(vis_g != vis_r)
    if len(diff):
        assert _knife_edge(wl, idx, diff).all(), f"{len(diff)} mask mismatches off the depth knife edge"
        ok_rows = np.setdiff1d(np.arange(len(idx)), diff[:, 0])
    else:
        ok_rows = np.arange(len(idx))
    assert np.array_equal(g["counts"][idx][ok_rows], ref["counts"][ok_rows])
    assert np.array_equal(g["codes"][idx], ref["codes"])
    feat = (ref["counts"] > 0)[ok_rows]
    pg, pr = g["props"][idx][ok_rows][feat], ref["props"][ok_rows][feat]
    # density: relative; hardness (values in [0, 1]): relative to the property range
    rel_d = np.abs(pg[:, 0] - pr[:, 0]) / np.abs(pr[:, 0])
    err_h = np.abs(pg[:, 1] - pr[:, 1]) / np.abs(wl.values[:, 1]).max()
    assert rel_d.max() <= TOL_BF16, rel_d.max()
    assert err_h.max() <= TOL_BF16, err_h.max()
    assert (g["props"][idx][ok_rows][~feat] == 0).all()
    return rel_d, err_h


def test_c3_full_object_vs_oracle(cuda):
    from paper_2511_03126_b200 import workloads

    wl = workloads.generate("c3", device_splat=True)
    g = _gpu_full(wl)
    ref = oracle_rows(wl)
    rel_d, _ = _check_rows(wl, g, ref)
    mass_ref, occ_ref = O.voxel_mass(ref["codes"], ref["props"][:, 0], ref["edge"])
    assert g["mass"] == pytest.approx(mass_ref, rel=TOL_BF16)
    np.testing.assert_allclose(g["partials"]["weight_totals"], ref["weight_totals"], rtol=TOL_BF16)
    wt_rel = np.abs(g["partials"]["weight_totals"] - ref["weight_totals"]) / np.abs(ref["weight_totals"])
    assert g["partials"]["featured"] == int((ref["counts"] > 0).sum())
    print(f"C3 full object: density max rel {rel_d.max():.2e} (mean {rel_d.mean():.2e}), "
          f"mass {g['mass']:.6f} vs {mass_ref:.6f}, weight totals max rel {wt_rel.max():.2e}")


def test_c5_full_object_vs_oracle_slice(cuda):
    from paper_2511_03126_b200 import workloads

    wl = workloads.generate("c5", device_splat=True)
    g = _gpu_full(wl)
    idx = np.arange(0, wl.cfg.n, 8)
    ref = oracle_rows(wl, idx)
    rel_d, _ = _check_rows(wl, g, ref)
    print(f"C5 full object, {len(idx)}-point slice: density max rel {rel_d.max():.2e} (mean {rel_d.mean():.2e})")


def test_simt_bf16_d1024_c5_shape_vs_oracle(cuda, workload):
    """k_fuse_simt<1, 8, 4> (bf16 maps, D = 1024: the SIMT overflow kernel of C3 / C5) at the fp32 bar:
    it accumulates the exactly upcast bf16 values in fp32."""
    from test_gpu_fused import TOL, assert_parity, run_gpu, run_oracle

    wl = workload("c5", n=24_000)
    assert_parity(run_gpu(wl, force_simt=True), run_oracle(wl), wl, tol=TOL)
