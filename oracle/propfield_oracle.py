"""CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function cites the reference (`/root/reference/pkg/src/propfield/...`) line range it
restates. Arithmetic is float64 numpy in the reference's operation order. The two hot loops
(`visible_in_view`, `accumulate_features`) are also restated as numba `@njit` loops with fastmath
off, mirroring the reference's shipped numba backend (numba_impl.py:15-89), so the timed CPU
baseline runs at the reference's own speed; both builds agree bit for bit with the numpy forms.
"""

from __future__ import annotations

import math

import numpy as np

try:  # the reference's numba backend is optional there too (kernels/__init__.py:30-36)
    from numba import njit

    HAVE_NUMBA = True
except ImportError:  # pragma: no cover
    HAVE_NUMBA = False

    def njit(*a, **k):
        def wrap(f):
            return f

        return wrap if not (a and callable(a[0])) else a[0]


class PropfieldError(Exception):
    """errors.py:4-5 (restated so the oracle raises the reference's classes without importing the
    product package)."""


class MaterialError(PropfieldError):
    """errors.py:24-25: softmax_weights raises it on NaN similarities (grounding.py:173-174)."""


# ---- geometry -----------------------------------------------------------------------------------
def project_points(points, rotation, translation, fx, fy, cx, cy):
    """geometry.py:46-59: cam = p @ R.T + t; u = fx X / z + cx; v = fy Y / z + cy."""
    p = np.atleast_2d(np.asarray(points, dtype=np.float64))
    cam = p @ np.asarray(rotation, dtype=np.float64).T + np.asarray(translation, dtype=np.float64)
    z = cam[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        u = fx * cam[:, 0] / z + cx
        v = fy * cam[:, 1] / z + cy
    return u, v, z


def visible_in_view_np(u, v, z, depth_map, eps):
    """numpy_impl.py:14-40 (nearest pixel via round-half-even rint)."""
    h, w = depth_map.shape
    iu = np.rint(u).astype(np.int64)
    iv = np.rint(v).astype(np.int64)
    ok = (z > 0.0) & (iu >= 0) & (iu < w) & (iv >= 0) & (iv < h)
    out = np.zeros(u.shape[0], dtype=np.bool_)
    idx = np.flatnonzero(ok)
    if idx.size == 0:
        return out
    stored = depth_map[iv[idx], iu[idx]].astype(np.float64)
    out[idx] = (stored > 0.0) & (z[idx] <= stored + eps)
    return out


@njit(cache=True)
def _visible_in_view_nb(u, v, z, depth_map, eps):
    """numba_impl.py:15-32 restated."""
    h, w = depth_map.shape
    n = u.shape[0]
    iu = np.rint(u)
    iv = np.rint(v)
    out = np.zeros(n, dtype=np.bool_)
    for i in range(n):
        if z[i] <= 0.0:
            continue
        x = int(iu[i])
        y = int(iv[i])
        if x < 0 or x >= w or y < 0 or y >= h:
            continue
        stored = float(depth_map[y, x])
        if stored > 0.0 and z[i] <= stored + eps:
            out[i] = True
    return out


def visible_in_view(u, v, z, depth_map, eps, impl="numba"):
    if impl == "numba" and HAVE_NUMBA:
        return _visible_in_view_nb(np.ascontiguousarray(u, np.float64), np.ascontiguousarray(v, np.float64),
                                   np.ascontiguousarray(z, np.float64),
                                   np.ascontiguousarray(depth_map, np.float32), float(eps))
    return visible_in_view_np(u, v, z, depth_map, eps)


def visibility_mask(points, views, epsilon, impl="numba"):
    """geometry.py:89-103: per view, project then depth-test."""
    p = np.atleast_2d(np.asarray(points, dtype=np.float64))
    mask = np.zeros((p.shape[0], len(views)), dtype=np.bool_)
    for j, view in enumerate(views):
        u, v, z = project_points(p, view.camera.rotation, view.camera.translation,
                                 view.intrinsics.fx, view.intrinsics.fy, view.intrinsics.cx,
                                 view.intrinsics.cy)
        mask[:, j] = visible_in_view(u, v, z, np.asarray(view.depth, np.float32), epsilon, impl)
    return mask


# ---- bilinear gather / accumulation ------------------------------------------------------------------
def bilinear_gather(fmap, fu, fv):
    """numpy_impl.py:43-66: border-clamped bilinear, float64 (M, D)."""
    h, w, _ = fmap.shape
    x = np.clip(fu, 0.0, w - 1.0)
    y = np.clip(fv, 0.0, h - 1.0)
    x0 = np.floor(x).astype(np.int64)
    y0 = np.floor(y).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    wx = (x - x0)[:, None]
    wy = (y - y0)[:, None]
    f00 = fmap[y0, x0].astype(np.float64)
    f01 = fmap[y0, x1].astype(np.float64)
    f10 = fmap[y1, x0].astype(np.float64)
    f11 = fmap[y1, x1].astype(np.float64)
    return (
        f00 * ((1.0 - wy) * (1.0 - wx))
        + f01 * ((1.0 - wy) * wx)
        + f10 * (wy * (1.0 - wx))
        + f11 * (wy * wx)
    )


@njit(cache=True)
def _accumulate_nb(fmap, fu, fv, rows, accum, counts):
    """numba_impl.py:63-89 restated (serial loop over samples and channels)."""
    h, w, dim = fmap.shape
    m = fu.shape[0]
    for i in range(m):
        x = min(max(fu[i], 0.0), w - 1.0)
        y = min(max(fv[i], 0.0), h - 1.0)
        x0 = int(math.floor(x))
        y0 = int(math.floor(y))
        x1 = min(x0 + 1, w - 1)
        y1 = min(y0 + 1, h - 1)
        wx = x - x0
        wy = y - y0
        w00 = (1.0 - wy) * (1.0 - wx)
        w01 = (1.0 - wy) * wx
        w10 = wy * (1.0 - wx)
        w11 = wy * wx
        r = rows[i]
        for d in range(dim):
            val = (
                fmap[y0, x0, d] * w00
                + fmap[y0, x1, d] * w01
                + fmap[y1, x0, d] * w10
                + fmap[y1, x1, d] * w11
            )
            accum[r, d] = accum[r, d] + val
        counts[r] += 1


def accumulate_features(fmap, fu, fv, rows, accum, counts, impl="numba"):
    """numpy_impl.py:69-77 / numba_impl.py:63-89: accum[rows] += sample, counts[rows] += 1."""
    if impl == "numba" and HAVE_NUMBA:
        _accumulate_nb(np.ascontiguousarray(fmap, np.float32), np.ascontiguousarray(fu, np.float64),
                       np.ascontiguousarray(fv, np.float64), np.ascontiguousarray(rows, np.int64),
                       accum, counts)
        return
    sampled = bilinear_gather(fmap, fu, fv)
    accum[rows] += sampled
    counts[rows] += 1


def aggregate_geometric_features(positions, views, visibility, impl="numba"):
    """fusion.py:65-93: visibility-masked mean of bilinear samples; zero rows stay featureless.

    Returns (features (N,D) f64, visible_counts (N,) int64)."""
    p = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    n = p.shape[0]
    dim = int(views[0].feature_map.shape[2])
    accum = np.zeros((n, dim), dtype=np.float64)
    counts = np.zeros(n, dtype=np.int64)
    for j, view in enumerate(views):
        rows = np.flatnonzero(visibility[:, j])
        if rows.size == 0:
            continue
        u, v, _ = project_points(p[rows], view.camera.rotation, view.camera.translation,
                                 view.intrinsics.fx, view.intrinsics.fy, view.intrinsics.cx,
                                 view.intrinsics.cy)
        h, w = view.depth.shape
        fm = np.asarray(view.feature_map, dtype=np.float32)
        hf, wf, _ = fm.shape
        fu = (u + 0.5) * (wf / w) - 0.5
        fv = (v + 0.5) * (hf / h) - 0.5
        accumulate_features(fm, fu, fv, rows.astype(np.int64), accum, counts, impl)
    nonzero = counts > 0
    accum[nonzero] /= counts[nonzero, None]
    return accum, counts


# ---- normalisation + grounding --------------------------------------------------------------------
def normalize_rows(features):
    """Rule of fusion.py:210-214: f / |f| when |f| > 0, zero vectors stay zero."""
    f = np.asarray(features, dtype=np.float64)
    norm = np.linalg.norm(f, axis=1, keepdims=True)
    out = np.zeros_like(f)
    nz = norm[:, 0] > 0
    out[nz] = f[nz] / norm[nz]
    return out


def material_similarity(features, text_embeddings):
    """grounding.py:158-165: plain dot product of unit vectors, (S, K)."""
    f = np.atleast_2d(np.asarray(features, dtype=np.float64))
    return f @ np.asarray(text_embeddings, dtype=np.float64).T


def softmax_weights(similarities, temperature):
    """grounding.py:168-178."""
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    sims = np.atleast_2d(np.asarray(similarities, dtype=np.float64))
    if np.isnan(sims).any():
        raise MaterialError("NaN similarity passed to kernel regression")
    scaled = sims / temperature
    scaled -= scaled.max(axis=1, keepdims=True)
    w = np.exp(scaled)
    return w / w.sum(axis=1, keepdims=True)


def regress_with_weights(weights, values):
    """grounding.py:198-202."""
    w = np.atleast_2d(np.asarray(weights, dtype=np.float64))
    return w @ np.asarray(values, dtype=np.float64)


# ---- voxel-grid mass (BASELINE-defined; parity UNPINNED) --------------------------------------------
def voxel_domain(points):
    """Per-axis bbox of the f32 points, upcast exactly to f64 -> (lo (3,), hi (3,))."""
    p = np.asarray(points, dtype=np.float64)
    return p.min(axis=0), p.max(axis=0)


def voxel_codes(points, grid, lo=None, hi=None):
    """sampling.py:110-123 convention: cell = clip(floor((p - lo) / edge), 0, G-1),
    code = (cx*G + cy)*G + cz with edge = max extent / G. Returns (codes int64, edge)."""
    p = np.asarray(points, dtype=np.float64)
    if lo is None or hi is None:
        lo, hi = voxel_domain(p)
    edge = float((np.asarray(hi) - np.asarray(lo)).max()) / grid
    if edge > 0:
        cell = np.clip(np.floor((p - lo) / edge), 0, grid - 1).astype(np.int64)
    else:
        cell = np.zeros_like(p, dtype=np.int64)
    codes = (cell[:, 0] * grid + cell[:, 1]) * grid + cell[:, 2]
    return codes, edge


def voxel_mass(codes, rho, edge):
    """mass = edge^3 * sum over occupied voxels of the mean point density (1-voxel shell)."""
    codes = np.asarray(codes, dtype=np.int64)
    uniq, inv = np.unique(codes, return_inverse=True)
    sums = np.bincount(inv, weights=np.asarray(rho, dtype=np.float64))
    cnt = np.bincount(inv)
    return float(edge**3 * np.sum(sums / cnt)), int(uniq.size)


# ---- integrate_mass partials (integrate.py:98-167) ---------------------------------------------------
def integrate_partials(weights, positions, mid_density, theta, normals=None):
    """The data-parallel part of integrate_mass: weight_totals (integrate.py:133), point mass
    pm_i = w_i @ (mid * theta) (integrate.py:146, without lam*b^2), sum pm, sum pm * centre with
    centre = position - (w_i @ theta / 2) * normal when normals are given (integrate.py:149-152)."""
    w = np.asarray(weights, dtype=np.float64)
    pm = w @ (np.asarray(mid_density, np.float64) * np.asarray(theta, np.float64))
    pos = np.asarray(positions, dtype=np.float64)
    if normals is not None:
        mean_theta = w @ np.asarray(theta, np.float64)
        pos = pos - (mean_theta[:, None] / 2.0) * np.asarray(normals, np.float64)
    return {
        "weight_totals": w.sum(axis=0),
        "pm_sum": float(pm.sum()),
        "pm_pos": (pm[:, None] * pos).sum(axis=0),
    }


def characteristic_length(positions, k=8):
    """integrate.py:72-95 (k-th neighbour area estimate; bbox fallback below 4 points)."""
    from scipy.spatial import cKDTree

    p = np.asarray(positions, dtype=np.float64)
    n = p.shape[0]
    if n == 0:
        return 0.0
    if n < 4:
        return float((p.max(axis=0) - p.min(axis=0)).max())
    k_eff = min(k, n - 1)
    dist, _ = cKDTree(p).query(p, k=k_eff + 1)
    d_k = dist[:, k_eff]
    return float(np.sqrt(np.pi / k_eff * np.sum(d_k * d_k)))


# ---- the north-star composition ---------------------------------------------------------
def fuse_and_query(points, views, text, values, temperature, epsilon, grid, density_col=0,
                   mid_theta=None, impl="numba"):
    """visibility -> aggregate -> normalise -> similarity -> softmax -> regress -> voxel mass.

    Featureless points (count 0) get all-zero probability and property rows (pipeline.py:279-280)
    and still occupy their voxel with rho = 0."""
    p = np.asarray(points, dtype=np.float64)
    vis = visibility_mask(p, views, epsilon, impl)
    feats, counts = aggregate_geometric_features(p, views, vis, impl)
    fhat = normalize_rows(feats)
    featured = counts > 0
    k = np.asarray(text).shape[0]
    sims = np.zeros((p.shape[0], k))
    weights = np.zeros((p.shape[0], k))
    if featured.any():
        sims[featured] = material_similarity(fhat[featured], text)
        weights[featured] = softmax_weights(sims[featured], temperature)
    props = regress_with_weights(weights, values)
    codes, edge = voxel_codes(points, grid)
    mass, occupied = voxel_mass(codes, props[:, density_col], edge)
    out = {
        "visibility": vis,
        "counts": counts,
        "features": feats,
        "fhat": fhat,
        "sims": sims,
        "weights": weights,
        "props": props,
        "codes": codes,
        "edge": edge,
        "mass": mass,
        "occupied": occupied,
    }
    if mid_theta is not None:
        out.update(integrate_partials(weights, p, mid_theta, np.ones_like(mid_theta)))
    return out


# ---- densification ---------------------------------------------------------------
def dino_knn_interpolate(query_features, source_features, source_probs, k):
    """densify.py:36-86: cosine k-NN in feature space, neighbours by (-sim, index), weights
    max(sim, 0) renormalised (uniform 1/k when they all vanish), convex combination of the
    neighbours' probability rows. Zero query rows raise ValueError-compatible MaterialError text."""
    q = np.atleast_2d(np.asarray(query_features, dtype=np.float64))
    s = np.atleast_2d(np.asarray(source_features, dtype=np.float64))
    probs = np.atleast_2d(np.asarray(source_probs, dtype=np.float64))
    if k < 1 or k > s.shape[0]:
        raise ValueError(f"k={k} outside 1..{s.shape[0]}")
    qn = np.linalg.norm(q, axis=1)
    missing = np.flatnonzero(qn == 0)
    if missing.size:
        raise ValueError(f"query features missing for indices {missing[:10].tolist()}")
    su = s / np.maximum(np.linalg.norm(s, axis=1, keepdims=True), 1e-30)
    sims = (q / qn[:, None]) @ su.T
    # full lexicographic order (-sim, index) per row, first k (densify.py:69-76)
    idx = np.broadcast_to(np.arange(s.shape[0]), sims.shape)
    order = np.lexsort((idx, -sims), axis=1)[:, :k]
    nsims = np.take_along_axis(sims, order, axis=1)
    w = np.maximum(nsims, 0.0)
    tot = w.sum(axis=1)
    flat = tot <= 0
    w[flat] = 1.0
    tot[flat] = k
    w /= tot[:, None]
    return np.einsum("qk,qkm->qm", w, probs[order])


def densify_field(positions, features, visible_counts, source_features, source_probs, values_by_prop, k):
    """densify.py:110-160: featured points interpolate in feature space; featureless ones (count 0
    or zero feature row) copy their nearest featured neighbour's probabilities (brute-force fp64
    nearest, lowest index on ties — the cKDTree k=1 query); properties regress the probabilities
    on each property's [lo, hi] table (one column when lo == hi). Returns a dict."""
    pos = np.asarray(positions, dtype=np.float64)
    f = np.asarray(features, dtype=np.float64)
    n = pos.shape[0]
    k = min(k, np.asarray(source_features).shape[0])
    featureless = (np.asarray(visible_counts) == 0) | (np.linalg.norm(f, axis=1) == 0)
    m = np.asarray(source_probs).shape[1]
    probs = np.zeros((n, m))
    featured = np.flatnonzero(~featureless)
    if featured.size:
        probs[featured] = dino_knn_interpolate(f[featured], source_features, source_probs, k)
    orphan = np.flatnonzero(featureless)
    if orphan.size:
        if featured.size == 0:
            raise ValueError("no point in the cloud has a geometric feature")
        fp = pos[featured]
        for i in orphan:
            d2 = ((fp - pos[i]) ** 2).sum(axis=1)
            probs[i] = probs[featured[int(np.argmin(d2))]]
    props = {}
    for name, lo_hi in values_by_prop.items():
        lo_hi = np.asarray(lo_hi, dtype=np.float64)
        props[name] = regress_with_weights(probs, lo_hi[:, 0] if np.all(lo_hi[:, 0] == lo_hi[:, 1]) else lo_hi)
    return {"probabilities": probs, "dominant": probs.argmax(axis=1), "properties": props,
            "featureless": featureless}


# ---- normals -----------------------------------------------------------------------
def estimate_normals(positions, k, camera_centers):
    """geometry.py:106-146: cKDTree k-NN (self included), neighbourhood covariance / k
    (numpy_impl.py:115-128), eigh, smallest eigenvector, rank < 2 fallback to the camera direction
    (ratio 1e-10, geometry.py:13), orientation toward the mean camera centre."""
    from scipy.spatial import cKDTree

    p = np.asarray(positions, dtype=np.float64)
    n = p.shape[0]
    if k < 3:
        raise ValueError(f"normal estimation needs k >= 3, got {k}")
    if k > n:
        raise ValueError(f"k={k} exceeds point count {n}")
    _, nb = cKDTree(p).query(p, k=k)
    q = p[nb]
    mu = q.sum(axis=1) / q.shape[1]
    d = q - mu[:, None, :]
    cov = np.einsum("nki,nkj->nij", d, d) / q.shape[1]
    w, v = np.linalg.eigh(cov)
    normals = np.ascontiguousarray(v[:, :, 0])
    to_cam = np.asarray(camera_centers, dtype=np.float64).mean(axis=0) - p
    degenerate = w[:, 1] <= 1e-10 * np.maximum(w[:, 2], 1e-300)
    if degenerate.any():
        fb = to_cam[degenerate]
        normals[degenerate] = fb / np.maximum(np.linalg.norm(fb, axis=1, keepdims=True), 1e-30)
    flip = np.einsum("ij,ij->i", normals, to_cam) < 0
    normals[flip] *= -1.0
    normals /= np.maximum(np.linalg.norm(normals, axis=1, keepdims=True), 1e-30)
    return normals, degenerate
