"""Operator- and function-level drop-in API on the GPU vs the reference's golden vectors.

Bar: bit-exact (rtol = atol = 0), as the reference's own cross-backend test demands
(tests/test_kernels.py:19-57), for masks, gathers, accumulations, aggregated features; the f64
similarity GEMM within 1e-13 (BLAS summation order differs).
"""

import hashlib

import numpy as np
import pytest

import recipes
import paper_2511_03126_b200 as pf
from paper_2511_03126_b200 import kernels
from paper_2511_03126_b200.errors import MaterialError

pytestmark = pytest.mark.gpu


def simple_view(w=64, h=64, fx=100.0, fy=100.0, cx=None, cy=None, depth_value=2.0,
                feature_size=(8, 8), feature_dim=4, fmap=None):
    """Identity-pose view with a constant depth plane (reference tests/conftest.py:70-88)."""
    return pf.ViewRecord(
        depth=np.full((h, w), depth_value, dtype=np.float32),
        camera=pf.CameraPose(rotation=np.eye(3), translation=np.zeros(3)),
        intrinsics=pf.Intrinsics(fx=fx, fy=fy, cx=cx if cx is not None else w / 2,
                                 cy=cy if cy is not None else h / 2),
        feature_map=fmap if fmap is not None else np.zeros((*feature_size, feature_dim), np.float32),
    )


class TestKernelRegistry:
    def test_visible_in_view_bit_exact(self, cuda, golden):
        g = golden("kernels")
        u, v, z, depth = recipes.visible_case()
        assert np.array_equal(np.packbits(kernels.visible_in_view(u, v, z, depth, 0.0)), g["visible_eps0"])
        assert np.array_equal(np.packbits(kernels.visible_in_view(u, v, z, depth, 0.05)), g["visible_eps005"])

    def test_bilinear_gather_bit_exact(self, cuda, golden):
        fmap, fu, fv = recipes.gather_case()
        np.testing.assert_allclose(kernels.bilinear_gather(fmap, fu, fv), golden("kernels")["gather"],
                                   rtol=0, atol=0)

    def test_accumulate_in_place_bit_exact(self, cuda, golden):
        g = golden("kernels")
        fmap, fu, fv, rows = recipes.accumulate_case()
        acc = np.zeros((300, 4))
        cnt = np.zeros(300, dtype=np.int64)
        assert kernels.accumulate_features(fmap, fu, fv, rows, acc, cnt) is None
        np.testing.assert_allclose(acc, g["accum"], rtol=0, atol=0)
        assert np.array_equal(cnt, g["accum_counts"])

    def test_accumulate_torch_stays_on_device(self, cuda, golden):
        import torch

        g = golden("kernels")
        fmap, fu, fv, rows = recipes.accumulate_case()
        acc = torch.zeros((300, 4), dtype=torch.float64, device=cuda)
        cnt = torch.zeros(300, dtype=torch.int64, device=cuda)
        kernels.accumulate_features(torch.from_numpy(fmap).cuda(), torch.from_numpy(fu).cuda(),
                                    torch.from_numpy(fv).cuda(), torch.from_numpy(rows).cuda(), acc, cnt)
        assert acc.is_cuda
        np.testing.assert_allclose(acc.cpu().numpy(), g["accum"], rtol=0, atol=0)

    def test_bf16_map_equals_upcast_f32(self, cuda):
        from paper_2511_03126_b200.workloads import bf16_bits_to_f32, f32_to_bf16_bits

        fmap, fu, fv = recipes.gather_case()
        bits = f32_to_bf16_bits(fmap)
        a = kernels.bilinear_gather(bits, fu, fv)
        b = kernels.bilinear_gather(bf16_bits_to_f32(bits), fu, fv)
        np.testing.assert_array_equal(a, b)

    def test_backend_is_cuda_only(self):
        assert kernels.available_backends() == ["cuda"]
        with pytest.raises(ValueError):
            kernels.set_backend("numba")

    def test_empty_inputs(self, cuda):
        out = kernels.visible_in_view(np.zeros(0), np.zeros(0), np.zeros(0),
                                      np.ones((4, 4), np.float32), 0.1)
        assert out.shape == (0,)
        g = kernels.bilinear_gather(np.ones((2, 2, 3), np.float32), np.zeros(0), np.zeros(0))
        assert g.shape == (0, 3)


class TestGeometry:
    """Known answers of the reference's tests/test_geometry.py:20-66."""

    def test_hand_computed_pinhole(self, cuda):
        view = simple_view(fx=100, fy=100, cx=50, cy=50)
        pix, z = pf.project_points(np.array([[1.0, 0.0, 2.0]]), view.camera, view.intrinsics)
        assert np.allclose(pix[0], [100.0, 50.0]) and z[0] == 2.0

    def test_on_surface_visible_behind_not(self, cuda):
        view = simple_view(depth_value=2.0)
        assert pf.visibility_mask(np.array([[0.0, 0.0, 2.0]]), [view], 0.0)[0, 0]
        assert not pf.visibility_mask(np.array([[0.0, 0.0, 3.0]]), [view], 0.0)[0, 0]

    def test_out_of_bounds_and_invalid_depth(self, cuda):
        v = simple_view(w=16, h=16, fx=10, fy=10, cx=8, cy=8)
        assert not pf.visibility_mask(np.array([[50.0, 0.0, 1.0]]), [v], 10.0)[0, 0]
        assert not pf.visibility_mask(np.array([[0.0, 0.0, 1.0]]), [simple_view(depth_value=0.0)], 10.0)[0, 0]
        # behind the camera
        assert not pf.visibility_mask(np.array([[0.0, 0.0, -1.0]]), [simple_view()], 10.0)[0, 0]

    def test_half_pixel_rounds_to_even(self, cuda):
        # u = 100 * x / 2 + 32 = 31.5 -> rint -> 32 (even); depth 0 at column 31, valid at 32
        view = simple_view(fx=100, fy=100, cx=32, cy=32)
        view.depth[:, 31] = 0.0
        x = (31.5 - 32.0) * 2.0 / 100.0
        assert pf.visibility_mask(np.array([[x, 0.0, 2.0]]), [view], 0.0)[0, 0]

    @pytest.mark.parametrize("name", ["mini", "mini_bf16"])
    def test_mask_bit_exact_vs_reference(self, cuda, golden, workload, name):
        g = golden(name)
        wl = workload(name)
        vis = pf.visibility_mask(wl.points.astype(np.float64), wl.views(), wl.cfg.eps)
        ref = np.unpackbits(g["visibility"], axis=1)[:, : wl.cfg.nviews].astype(bool)
        assert np.array_equal(vis, ref)

    def test_mask_scale_invariance(self, cuda, workload):
        """tests/test_geometry.py:217-228: scaling the scene and eps together keeps the mask."""
        wl = workload("mini")
        p = wl.points.astype(np.float64)
        vis = pf.visibility_mask(p, wl.views(), wl.cfg.eps)
        scaled = []
        for v in wl.views():
            cam = pf.CameraPose(rotation=v.camera.rotation, translation=v.camera.translation * 2.0)
            scaled.append(pf.ViewRecord(depth=v.depth * 2.0, camera=cam, intrinsics=v.intrinsics,
                                        feature_map=v.feature_map))
        vis2 = pf.visibility_mask(p * 2.0, scaled, wl.cfg.eps * 2.0)
        assert np.array_equal(vis, vis2)


class TestFusion:
    def test_single_view_equals_sampled_feature(self, cuda):
        """tests/test_fusion.py:41-50."""
        rng = np.random.default_rng(0)
        fmap = rng.standard_normal((16, 16, 3)).astype(np.float32)
        view = simple_view(w=16, h=16, depth_value=2.0, fmap=fmap)
        pts = np.array([[0.0, 0.0, 2.0], [0.02, -0.01, 2.0]])
        sem = pf.aggregate_geometric_features(pts, [view], np.ones((2, 1), dtype=bool))
        pix, _ = pf.project_points(pts, view.camera, view.intrinsics)
        fu = (pix[:, 0] + 0.5) * (16 / 16) - 0.5
        fv = (pix[:, 1] + 0.5) * (16 / 16) - 0.5
        assert np.array_equal(sem.features, kernels.bilinear_gather(fmap, fu, fv))

    def test_zero_visible_points_flagged(self, cuda):
        view = simple_view(depth_value=1.0)
        sem = pf.aggregate_geometric_features(np.array([[0.0, 0.0, 0.5], [0.0, 0.0, 5.0]]), [view],
                                              np.array([[True], [False]]))
        assert not sem.featureless[0] and sem.featureless[1]
        assert np.all(sem.features[1] == 0)

    @pytest.mark.parametrize("name", ["mini", "mini_bf16"])
    def test_features_bit_exact_vs_reference(self, cuda, golden, workload, name):
        g = golden(name)
        wl = workload(name)
        p = wl.points.astype(np.float64)
        vis = np.unpackbits(g["visibility"], axis=1)[:, : wl.cfg.nviews].astype(bool)
        sem = pf.aggregate_geometric_features(p, wl.views(), vis)
        assert np.array_equal(sem.visible_counts, g["counts"])
        assert hashlib.sha256(sem.features.tobytes()).hexdigest() == str(g["features_sha"])


class TestGrounding:
    @pytest.mark.parametrize("seed", [0, 1])
    def test_vs_reference(self, cuda, golden, seed):
        g = golden("grounding")
        f, t, y = recipes.grounding_case(seed)
        s = pf.material_similarity(f, t)
        np.testing.assert_allclose(s, g[f"sims{seed}"], rtol=0, atol=1e-13)
        w = pf.softmax_weights(s, 0.1)
        np.testing.assert_allclose(w, g[f"weights{seed}"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(pf.regress_with_weights(w, y), g[f"props{seed}"], rtol=1e-12)
        np.testing.assert_allclose(pf.kernel_regress(s, y[:, 0], 0.05), g[f"kreg{seed}"], rtol=1e-12)

    def test_known_answers(self, cuda):
        """tests/test_grounding.py:89-200."""
        assert pf.kernel_regress(np.array([[0.3]]), np.array([42.0]), 0.1)[0] == 42.0
        out = pf.kernel_regress(np.array([[0.5, 0.5]]), np.array([10.0, 30.0]), 0.1)
        assert out[0] == pytest.approx(20.0, abs=1e-12)
        rng = np.random.default_rng(0)
        sims = rng.uniform(-1, 1, size=(50, 5))
        vals = rng.uniform(0, 100, size=5)
        assert np.abs(pf.kernel_regress(sims, vals, 0.001) - vals[np.argmax(sims, 1)]).max() < 1e-6
        assert np.isfinite(pf.kernel_regress(np.array([[1.0, -1.0]]), np.array([5.0, 7.0]), 1e-4)).all()
        w = pf.softmax_weights(rng.uniform(-1, 1, (100, 4)), 0.1)
        assert np.all(w >= 0) and np.allclose(w.sum(1), 1.0)
        assert np.allclose(pf.material_similarity(np.array([[1.0, 0, 0]]), np.eye(3))[0], [1, 0, 0])

    def test_errors(self, cuda):
        with pytest.raises(MaterialError, match="NaN"):
            pf.kernel_regress(np.array([[np.nan, 0.0]]), np.array([1.0, 2.0]), 0.1)
        with pytest.raises(ValueError):
            pf.softmax_weights(np.array([[0.1]]), 0.0)


class TestVoxelMass:
    def test_codes_bit_exact(self, cuda, workload):
        from oracle import propfield_oracle as O

        wl = workload("mini")
        rho = np.random.default_rng(0).uniform(100, 8000, wl.cfg.n)
        mass, occ, codes = pf.voxel_mass(wl.points, rho, 32)
        ref_codes, edge = O.voxel_codes(wl.points, 32)
        assert np.array_equal(codes, ref_codes)
        ref_mass, ref_occ = O.voxel_mass(ref_codes, rho.astype(np.float32), edge)
        assert occ == ref_occ
        assert mass == pytest.approx(ref_mass, rel=1e-5)


class TestTensorCorePlumbing:
    @pytest.mark.parametrize("ts", [0, 1])
    @pytest.mark.parametrize("k,n", [(64, 128), (128, 128), (256, 64), (192, 128), (64, 16)])
    def test_umma_selftest_matches_matmul(self, cuda, k, n, ts):
        import torch

        from paper_2511_03126_b200 import _lib

        g = torch.Generator(device="cuda").manual_seed(k * 1000 + n)
        a = torch.randn(128, k, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(k, n, device="cuda", generator=g).to(torch.bfloat16)
        c = torch.empty(128, n, device="cuda", dtype=torch.float32)
        _lib.call("pf_selftest_umma", a.data_ptr(), b.data_ptr(), c.data_ptr(), k, n, ts,
                  torch.cuda.current_stream().cuda_stream)
        ref = a.float() @ b.float()
        torch.testing.assert_close(c, ref, rtol=1e-5, atol=1e-4)
