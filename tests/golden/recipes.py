"""Seeded input recipes shared by the golden-vector generator and the tests.

The operator recipes reproduce the reference's own cross-backend test inputs
(/root/reference/pkg/tests/test_kernels.py:19-57) draw for draw, so the golden outputs pin our
kernels to exactly the cases the reference pins its numba build with.
"""

import numpy as np


def visible_case():
    """test_kernels.py:19-31."""
    rng = np.random.default_rng(0)
    depth = rng.uniform(0, 3, size=(64, 64)).astype(np.float32)
    depth[depth < 0.3] = 0.0
    n = 20_000
    u = rng.uniform(-10, 74, size=n)
    v = rng.uniform(-10, 74, size=n)
    z = rng.uniform(-0.5, 3.5, size=n)
    return u, v, z, depth


def gather_case():
    """test_kernels.py:33-41."""
    rng = np.random.default_rng(1)
    fmap = rng.standard_normal((32, 48, 8)).astype(np.float32)
    fu = rng.uniform(-2, 50, size=5000)
    fv = rng.uniform(-2, 34, size=5000)
    return fmap, fu, fv


def accumulate_case():
    """test_kernels.py:43-56."""
    rng = np.random.default_rng(2)
    fmap = rng.standard_normal((16, 16, 4)).astype(np.float32)
    rows = rng.permutation(300)[:200].astype(np.int64)
    fu = rng.uniform(0, 15, size=200)
    fv = rng.uniform(0, 15, size=200)
    return fmap, fu, fv, rows


def grounding_case(seed=0, s=64, d=32, k=8):
    rng = np.random.default_rng(100 + seed)
    f = rng.standard_normal((s, d))
    f /= np.linalg.norm(f, axis=1, keepdims=True)
    t = rng.standard_normal((k, d))
    t /= np.linalg.norm(t, axis=1, keepdims=True)
    y = np.stack([rng.uniform(100, 8000, k), rng.uniform(0, 1, k)], axis=1)
    return f, t, y


def densify_cases():
    """dino_knn_interpolate inputs: the reference's own test_densify.py:29-94 cases draw for draw,
    plus larger seeded cases (ties from duplicated sources, k == S, negative-similarity rows)."""
    cases = []
    rng = np.random.default_rng(0)  # test_k1_copies_nearest_source
    src_feat = rng.standard_normal((10, 4))
    src_probs = rng.dirichlet(np.ones(3), size=10)
    cases.append(("k1_copy", src_feat[4][None, :] * 2.0, src_feat, src_probs, 1))
    cases.append(("equal_sims", np.array([[1.0, 0.0]]), np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 1.0]]),
                  np.array([[1.0, 0.0], [0.0, 1.0], [0.5, 0.5]]), 2))
    for k in (1, 3, 7):  # test_matches_exhaustive_oracle
        rng = np.random.default_rng(42)
        src_feat = rng.standard_normal((40, 8))
        src_probs = rng.dirichlet(np.ones(4), size=40)
        queries = rng.standard_normal((200, 8))
        cases.append((f"exhaustive_k{k}", queries, src_feat, src_probs, k))
    cases.append(("all_negative", np.array([[-1.0, 0.0]]), np.array([[1.0, 0.0], [0.9, 0.1]]),
                  np.array([[1.0, 0.0], [0.0, 1.0]]), 2))
    rng = np.random.default_rng(3)  # test_rows_are_convex_combinations
    cases.append(("convex", rng.standard_normal((100, 6)), rng.standard_normal((30, 6)),
                  rng.dirichlet(np.ones(5), size=30), 4))
    rng = np.random.default_rng(4)  # test_exact_feature_match_is_in_neighbor_set
    src_feat = rng.standard_normal((20, 5))
    cases.append(("exact_match", src_feat[7][None], src_feat, np.eye(20), 3))
    # larger: pipeline-like anchors (S=150, k=5, D=64, M=16), duplicated sources (exact ties)
    rng = np.random.default_rng(11)
    s = rng.standard_normal((150, 64))
    s[100:110] = s[0:10]
    q = rng.standard_normal((3000, 64))
    q[:50] = s[:50] * rng.uniform(0.5, 2.0, (50, 1))
    p = rng.dirichlet(np.ones(16), size=150)
    cases.append(("anchors150_k5", q, s, p, 5))
    cases.append(("anchors150_kS", q[:200], s, p, 150))
    return cases


def densify_field_case(seed=0, n=1500, n_sources=60, noise=0.05, n_orphans=40):
    """densify_field inputs in the shape of test_densify.py:97-124 (striped two-part layout) with
    some featureless points (zero rows, count 0) that take their nearest featured neighbour."""
    rng = np.random.default_rng(seed)
    pts = np.zeros((n, 3))
    pts[:, 0] = rng.uniform(0, 1, size=n)
    pts[:, 1] = rng.uniform(0, 1, size=n)
    part = (np.floor(pts[:, 0] / 0.05).astype(int) % 2).astype(np.int64)
    feats = np.zeros((n, 2))
    feats[np.arange(n), part] = 1.0
    feats = feats + noise * rng.standard_normal(feats.shape)
    counts = np.ones(n, dtype=np.int64)
    orphans = rng.choice(n, size=n_orphans, replace=False)
    feats[orphans] = 0.0
    counts[orphans] = 0
    featured = np.setdiff1d(np.arange(n), orphans)
    src_pick = rng.choice(featured, size=n_sources, replace=False)
    density = np.array([[600.0, 600.0], [7800.0, 7800.0]])
    hardness = np.array([[0.2, 0.4], [0.8, 0.9]])
    return dict(positions=pts, features=feats, counts=counts, src_pick=src_pick,
                src_features=feats[src_pick], src_probs=np.eye(2)[part[src_pick]], density=density,
                hardness=hardness, part=part)


def normals_cases():
    """estimate_normals inputs (f32 clouds as the bundle stores them): an ellipsoid, a plane with a
    collinear strip (rank-1 neighbourhoods -> degenerate fallback), several k."""
    rng = np.random.default_rng(31)
    out = []
    u = rng.standard_normal((3000, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    ell = (u * np.array([0.4, 0.3, 0.2])).astype(np.float32)
    cams = np.array([[1.5, 0.0, 0.5], [-0.7, 1.3, 0.5], [-0.7, -1.3, 0.5]])
    out.append(("ellipsoid_k16", ell, cams, 16))
    out.append(("ellipsoid_k8", ell, cams, 8))
    plane = np.zeros((1200, 3), np.float32)
    plane[:1000, :2] = rng.uniform(-0.5, 0.5, (1000, 2))
    plane[1000:, 0] = np.linspace(2.0, 3.0, 200)  # an isolated line: rank-1 neighbourhoods
    out.append(("plane_line_k6", plane, cams, 6))
    return out
