"""Device integrate_mass pieces against the pinned CPU oracle:

* characteristic_length (integrate.py:72-95): exact k-NN on the device vs cKDTree (oracle), on the
  path's own clouds, clustered clouds with sparse outliers (shell expansion), exact duplicates, a
  regular lattice (distance ties), k other than AREA_KNN, and the n < 4 bbox fallback; rel 1e-9 (fp64
  distances from the same f32 coordinates; only the summation order differs);
* integrate_mass (integrate.py:98-167) with and without normals: partial sums on the device, host
  arithmetic in the reference order; rel 1e-9.
"""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from oracle import propfield_oracle as O
from paper_2511_03126_b200.integrate import estimate_from_partials

pytestmark = pytest.mark.gpu


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("name", ["mini", "pr1"])
def test_characteristic_length_on_path_clouds(workload, name):
    pts = workload(name).points
    assert rel(pf.characteristic_length(pts), O.characteristic_length(pts.astype(np.float64))) <= 1e-9


def test_characteristic_length_clusters_outliers_duplicates():
    rng = np.random.default_rng(3)
    a = rng.normal(0.0, 0.01, (5000, 3))
    b = rng.normal(0.5, 0.002, (3000, 3))
    out = rng.uniform(-2, 2, (40, 3))          # isolated points: their k-NN lies many cells away
    dup = a[:200].copy()                       # exact duplicates (zero distances)
    pts = np.concatenate([a, b, out, dup]).astype(np.float32)
    for k in (8, 3, 15):
        assert rel(pf.characteristic_length(pts, k), O.characteristic_length(pts.astype(np.float64), k)) <= 1e-9


def test_characteristic_length_lattice_and_small_n():
    g = np.stack(np.meshgrid(np.arange(30), np.arange(30), np.arange(3), indexing="ij"), -1).reshape(-1, 3)
    pts = (g * 0.01).astype(np.float32)        # many equal distances
    assert rel(pf.characteristic_length(pts), O.characteristic_length(pts.astype(np.float64))) <= 1e-9
    small = np.array([[0, 0, 0], [1, 0, 0], [0, 2, 0]], np.float32)
    assert pf.characteristic_length(small) == O.characteristic_length(small.astype(np.float64))
    five = np.random.default_rng(0).uniform(0, 1, (5, 3)).astype(np.float32)  # k_eff = n - 1 = 4
    assert rel(pf.characteristic_length(five), O.characteristic_length(five.astype(np.float64))) <= 1e-9


@pytest.mark.parametrize("with_normals", [False, True])
def test_integrate_mass_matches_oracle(workload, with_normals):
    wl = workload("pr1")
    n, k = wl.points.shape[0], wl.text.shape[0]
    rng = np.random.default_rng(7)
    w = rng.dirichlet(np.ones(k), size=n)
    normals = None
    if with_normals:
        v = rng.normal(size=(n, 3))
        normals = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float32)
    names = [f"m{i}" for i in range(k)]
    dens = np.stack([wl.values[:, 0] * 0.9, wl.values[:, 0] * 1.1], axis=1)
    theta = rng.uniform(0.002, 0.02, k)

    class Dict:
        def __init__(self):
            self.names = names

        def property_values(self, prop):
            assert prop == "density"
            return dens

        def thicknesses(self):
            return theta

    fld = pf.PropertyField(positions=wl.points, probabilities=w, dominant=w.argmax(1), properties={},
                           material_names=names, normals=normals)
    cfg = pf.IntegrationConfig(lam=0.6, scale_factor=1.0)
    got = pf.integrate_mass(fld, Dict(), cfg)
    mid = dens.mean(axis=1)
    part = O.integrate_partials(w, wl.points, mid, theta, normals)
    length = O.characteristic_length(wl.points.astype(np.float64))
    want = estimate_from_partials(part["weight_totals"], part["pm_sum"], part["pm_pos"], n, Dict(), cfg, length)
    assert rel(got.characteristic_length, want.characteristic_length) <= 1e-9
    assert rel(got.mass_kg, want.mass_kg) <= 1e-9
    assert all(rel(a, b) <= 1e-9 for a, b in zip(got.mass_range, want.mass_range))
    assert np.allclose(got.center_of_mass, want.center_of_mass, rtol=1e-9, atol=1e-12)
    for nm in names:
        assert rel(got.per_material[nm], want.per_material[nm]) <= 1e-9
