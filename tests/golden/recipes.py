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
