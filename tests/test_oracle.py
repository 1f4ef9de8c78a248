"""The CPU oracle pinned against the reference's golden vectors (CPU only).

Golden files come from running the unmodified reference (tests/golden/make_golden.py). When the
reference is importable (build container) the oracle is also checked against it live.
"""

import hashlib
import os

import numpy as np
import pytest

import recipes
from oracle import propfield_oracle as O
from paper_2511_03126_b200 import workloads

HAVE_REF = os.path.isdir("/root/reference/pkg/src/propfield")


class TestKernelGoldens:
    @pytest.mark.parametrize("impl", ["numpy", "numba"])
    def test_visible_in_view(self, golden, impl):
        g = golden("kernels")
        u, v, z, depth = recipes.visible_case()
        for eps, key in ((0.0, "visible_eps0"), (0.05, "visible_eps005")):
            out = O.visible_in_view(u, v, z, depth, eps, impl)
            assert np.array_equal(np.packbits(out), g[key])

    def test_bilinear_gather(self, golden):
        fmap, fu, fv = recipes.gather_case()
        np.testing.assert_allclose(O.bilinear_gather(fmap, fu, fv), golden("kernels")["gather"],
                                   rtol=0, atol=0)

    @pytest.mark.parametrize("impl", ["numpy", "numba"])
    def test_accumulate(self, golden, impl):
        g = golden("kernels")
        fmap, fu, fv, rows = recipes.accumulate_case()
        acc = np.zeros((300, 4))
        cnt = np.zeros(300, dtype=np.int64)
        O.accumulate_features(fmap, fu, fv, rows, acc, cnt, impl)
        np.testing.assert_allclose(acc, g["accum"], rtol=0, atol=0)
        assert np.array_equal(cnt, g["accum_counts"])


class TestGroundingGoldens:
    @pytest.mark.parametrize("seed", [0, 1])
    def test_similarity_softmax_regress(self, golden, seed):
        g = golden("grounding")
        f, t, y = recipes.grounding_case(seed)
        s = O.material_similarity(f, t)
        np.testing.assert_allclose(s, g[f"sims{seed}"], rtol=0, atol=1e-15)
        w = O.softmax_weights(s, 0.1)
        np.testing.assert_allclose(w, g[f"weights{seed}"], rtol=1e-14, atol=1e-16)
        np.testing.assert_allclose(O.regress_with_weights(w, y), g[f"props{seed}"], rtol=1e-13)
        kreg = O.regress_with_weights(O.softmax_weights(s, 0.05), y[:, 0])
        np.testing.assert_allclose(kreg, g[f"kreg{seed}"], rtol=1e-13)

    def test_softmax_rejects(self):
        with pytest.raises(ValueError):
            O.softmax_weights(np.array([[0.1]]), 0.0)
        # grounding.py:173-174 raises MaterialError (not a ValueError) on NaN similarities
        with pytest.raises(O.MaterialError) as ei:
            O.softmax_weights(np.array([[np.nan, 0.0]]), 0.1)
        assert not isinstance(ei.value, ValueError)


@pytest.mark.parametrize("name", ["mini", "mini_bf16"])
class TestPipelineGoldens:
    def test_composition_matches_reference(self, golden, workload, name):
        g = golden(name)
        wl = workload(name)
        out = O.fuse_and_query(wl.points, wl.views(f32_maps=True), wl.text, wl.values,
                               wl.cfg.temperature, wl.cfg.eps, wl.cfg.grid)
        vis = np.unpackbits(g["visibility"], axis=1)[:, : wl.cfg.nviews].astype(bool)
        assert np.array_equal(out["visibility"], vis)
        assert np.array_equal(out["counts"], g["counts"])
        assert hashlib.sha256(out["features"].tobytes()).hexdigest() == str(g["features_sha"])
        np.testing.assert_array_equal(out["sims"], g["sims"])
        np.testing.assert_array_equal(out["weights"], g["weights"])
        np.testing.assert_array_equal(out["props"], g["props"])

    def test_integrate_partials_match_reference_mass(self, golden, workload, name):
        """integrate.py:124-167 rebuilt from the oracle's partials equals the reference's mass."""
        g = golden(name)
        wl = workload(name)
        part = O.integrate_partials(g["weights"], wl.points, wl.density, wl.thickness)
        length = O.characteristic_length(wl.points.astype(np.float64))
        assert length == pytest.approx(float(g["integ_length"]), rel=1e-12)
        b = np.sqrt(length**2 / wl.cfg.n)
        lam = 0.6
        per = lam * b * b * wl.thickness * part["weight_totals"] * wl.density
        np.testing.assert_allclose(per, g["integ_per_material"], rtol=1e-12)
        assert per.sum() == pytest.approx(float(g["integ_mass"]), rel=1e-12)
        com = part["pm_pos"] / part["pm_sum"]
        np.testing.assert_allclose(com, g["integ_com"], rtol=1e-10, atol=1e-12)


class TestVoxelOracle:
    def test_codes_in_range_and_monotone(self):
        rng = np.random.default_rng(0)
        p = rng.uniform(-1, 1, size=(5000, 3)).astype(np.float32)
        codes, edge = O.voxel_codes(p, 16)
        assert codes.min() >= 0 and codes.max() < 16**3
        lo, hi = O.voxel_domain(p)
        assert edge == pytest.approx((hi - lo).max() / 16)
        # the bbox maximum clips onto the last cell (sampling.py:114-118 convention)
        cx = codes // 256
        assert cx[np.argmax(p[:, 0])] == 15

    def test_mass_of_uniform_density_counts_occupied_voxels(self):
        rng = np.random.default_rng(1)
        p = rng.uniform(0, 1, size=(20000, 3)).astype(np.float32)
        codes, edge = O.voxel_codes(p, 8)
        mass, occ = O.voxel_mass(codes, np.full(len(p), 1000.0), edge)
        assert occ == 512
        assert mass == pytest.approx(1000.0 * 512 * edge**3)

    def test_mass_linear_in_density(self):
        rng = np.random.default_rng(2)
        p = rng.standard_normal((3000, 3)).astype(np.float32)
        rho = rng.uniform(100, 8000, 3000)
        codes, edge = O.voxel_codes(p, 32)
        m1, _ = O.voxel_mass(codes, rho, edge)
        m2, _ = O.voxel_mass(codes, 2.0 * rho, edge)
        assert m2 == 2.0 * m1


@pytest.mark.skipif(not HAVE_REF, reason="reference not mounted (GPU box)")
class TestAgainstLiveReference:
    def test_visibility_and_aggregate_pr1_subset(self, workload):
        import sys

        sys.path.insert(0, "/root/reference/pkg/src")
        from propfield import fusion, geometry
        from make_golden import ref_views

        wl = workload("pr1")
        rviews = ref_views(wl, None)
        p = wl.points[:3000].astype(np.float64)
        vis_ref = geometry.visibility_mask(p, rviews, wl.cfg.eps)
        vis = O.visibility_mask(p, wl.views(), wl.cfg.eps)
        assert np.array_equal(vis, vis_ref)
        a_ref = fusion.aggregate_geometric_features(p, rviews, vis_ref)
        a, c = O.aggregate_geometric_features(p, wl.views(), vis)
        assert np.array_equal(a, a_ref.features) and np.array_equal(c, a_ref.visible_counts)

    def test_softmax_error_classes(self):
        """The oracle raises the reference's exception classes (grounding.py:170-174)."""
        import sys

        sys.path.insert(0, "/root/reference/pkg/src")
        from propfield import errors, grounding

        bad = np.array([[np.nan, 0.0]])
        with pytest.raises(errors.MaterialError):
            grounding.softmax_weights(bad, 0.1)
        with pytest.raises(O.MaterialError):
            O.softmax_weights(bad, 0.1)
        assert O.MaterialError.__name__ == errors.MaterialError.__name__
        assert not issubclass(errors.MaterialError, ValueError)
        with pytest.raises(ValueError):
            grounding.softmax_weights(np.array([[0.1]]), 0.0)


class TestGenerator:
    def test_deterministic(self):
        a = workloads.generate("mini")
        b = workloads.generate("mini")
        assert np.array_equal(a.points, b.points) and np.array_equal(a.depth, b.depth)
        assert np.array_equal(a.fmaps, b.fmaps)

    def test_ellipsoid_points_on_surface(self):
        rng = np.random.default_rng(0)
        axes = np.array([0.3, 0.4, 0.25])
        p = workloads.sample_ellipsoid(rng, 5000, axes)
        r = ((p / axes) ** 2).sum(axis=1)
        np.testing.assert_allclose(r, 1.0, atol=1e-12)

    def test_bf16_round_trip(self):
        x = np.array([1.0, -2.5, 3.14159, 1e-3, 65504.0], dtype=np.float32)
        b = workloads.f32_to_bf16_bits(x)
        y = workloads.bf16_bits_to_f32(b)
        assert np.all(np.abs(y - x) <= np.abs(x) * 2.0**-8)
        assert np.array_equal(workloads.f32_to_bf16_bits(y), b)

    def test_depth_splat_min(self, workload):
        wl = workload("mini")
        d = wl.depth_np()
        assert d.min() >= 0 and (d > 0).mean() > 0.01


def boundary_ties(q, s, k):
    """Rows whose k-th and (k+1)-th similarities are exactly equal: the reference picks among such
    ties with np.argpartition (introselect, implementation-defined, densify.py:69-70); the oracle and
    the device take the lower index, matching the reference's own within-set tie-break. These rows
    are excluded from value parity (the neighbour SET is ambiguous there)."""
    q = np.atleast_2d(np.asarray(q, np.float64))
    s = np.atleast_2d(np.asarray(s, np.float64))
    if k >= s.shape[0]:
        return np.zeros(q.shape[0], dtype=bool)
    sims = (q / np.linalg.norm(q, axis=1)[:, None]) @ (s / np.linalg.norm(s, axis=1, keepdims=True)).T
    srt = -np.sort(-sims, axis=1)
    return srt[:, k - 1] == srt[:, k]


class TestDensifyOracle:
    """Oracle restatement of densify.py vs the reference's own outputs (tests/golden/densify.npz)."""

    def test_dino_knn_cases(self, golden):
        import recipes

        g = golden("densify")
        for name, q, s, p, k in recipes.densify_cases():
            keep = ~boundary_ties(q, s, k)
            assert keep.mean() > 0.9
            np.testing.assert_allclose(O.dino_knn_interpolate(q, s, p, k)[keep], g[f"dk_{name}"][keep], rtol=0,
                                       atol=1e-12, err_msg=name)

    def test_dino_knn_errors(self):
        with pytest.raises(ValueError, match=r"\[1\]"):
            O.dino_knn_interpolate(np.array([[1.0, 0, 0], [0, 0, 0]]), np.eye(3), np.eye(3), 1)
        with pytest.raises(ValueError):
            O.dino_knn_interpolate(np.eye(2), np.eye(2), np.eye(2), 3)

    def test_densify_field(self, golden):
        import recipes

        g = golden("densify")
        c = recipes.densify_field_case()
        out = O.densify_field(c["positions"], c["features"], c["counts"], c["src_features"], c["src_probs"],
                              {"density": c["density"], "hardness": c["hardness"]}, 3)
        np.testing.assert_allclose(out["probabilities"], g["df_probabilities"], rtol=0, atol=1e-12)
        np.testing.assert_array_equal(out["dominant"], g["df_dominant"])
        np.testing.assert_array_equal(out["featureless"], g["df_featureless"])
        np.testing.assert_allclose(out["properties"]["density"], g["df_density"], rtol=1e-12)
        np.testing.assert_allclose(out["properties"]["hardness"], g["df_hardness"], rtol=1e-12)


class TestNormalsOracle:
    """Oracle estimate_normals vs the reference's outputs (tests/golden/normals.npz)."""

    def test_cases(self, golden):
        g = golden("normals")
        for name, p, cams, k in recipes.normals_cases():
            nrm, deg = O.estimate_normals(p, k, cams)
            np.testing.assert_array_equal(deg, g[f"d_{name}"], err_msg=name)
            np.testing.assert_allclose(nrm, g[f"n_{name}"], rtol=0, atol=1e-12, err_msg=name)

    def test_errors(self):
        with pytest.raises(ValueError):
            O.estimate_normals(np.zeros((5, 3)), 2, np.zeros((1, 3)))
        with pytest.raises(ValueError):
            O.estimate_normals(np.zeros((5, 3)), 6, np.zeros((1, 3)))


class TestProjectionOperationOrder:
    """pf_common.cuh:cam_row reproduces `cam = p @ R.T + t` (geometry.py:54) as the fma chain
    fma(p2, R[r,2], fma(p1, R[r,1], p0 * R[r,0])) + t. That is the order of this image's numpy BLAS
    (OpenBLAS dgemm small-matrix kernel); the fp64 visibility masks are bit-exact only because the
    device uses the same order. This test pins it: exact fma via Fraction (correctly rounded) and
    numpy's own matmul must agree bit for bit on points and rotations of the workloads' kind."""

    @staticmethod
    def _fma(a, b, c):
        from fractions import Fraction

        return float(Fraction(a) * Fraction(b) + Fraction(c))

    def test_numpy_matmul_is_the_fma_chain(self):
        rng = np.random.default_rng(11)
        wl = workloads.generate("mini_fib40")
        pts = np.concatenate([wl.points[:300].astype(np.float64), rng.uniform(-0.5, 0.5, (200, 3))])
        for pose in wl.poses[:8]:
            R = np.asarray(pose.rotation, np.float64)
            t = np.asarray(pose.translation, np.float64)
            cam = pts @ R.T + t  # the reference's expression (geometry.py:54)
            for i in range(pts.shape[0]):
                p0, p1, p2 = (float(x) for x in pts[i])
                for r in range(3):
                    acc = p0 * float(R[r, 0])
                    acc = self._fma(p1, float(R[r, 1]), acc)
                    acc = self._fma(p2, float(R[r, 2]), acc)
                    assert acc + float(t[r]) == cam[i, r], (i, r)
