"""Projection and depth-tested visibility (reference geometry.py:46-103), on the GPU.

`project_points` and `visibility_mask` keep the reference signatures and return the reference's
types (numpy in -> numpy out; torch CUDA in -> torch CUDA out). The fp64 arithmetic reproduces
numpy's rounding (see csrc/pf_common.cuh), so masks are bit-identical to the reference.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import ViewSet, cached_view_set, is_torch, ptr, require_cuda, stream_handle, to_dev, torch

DEFAULT_EPSILON_FRACTION = 0.01  # geometry.py:12


def _views_of(views, with_fmap: bool = True) -> ViewSet:
    return cached_view_set(views, with_fmap=with_fmap)


def project_points(points, camera, intrinsics):
    """Pinhole-project world points: ((N,2) pixels, (N,) z) float64 (geometry.py:46-59)."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(points)
    p = to_dev(points, t.float64, dev).reshape(-1, 3)
    rec = np.zeros(1, dtype=_lib.VIEW_DTYPE)
    rec["R"] = np.asarray(camera.rotation, dtype=np.float64).reshape(9)
    rec["t"] = np.asarray(camera.translation, dtype=np.float64)
    rec["fx"], rec["fy"] = intrinsics.fx, intrinsics.fy
    rec["cx"], rec["cy"] = intrinsics.cx, intrinsics.cy
    n = p.shape[0]
    uv = t.empty((n, 2), dtype=t.float64, device=dev)
    z = t.empty(n, dtype=t.float64, device=dev)
    _lib.call("pf_project_points", ptr(p), n, rec.ctypes.data, ptr(uv), ptr(z), stream_handle())
    return (uv, z) if tor else (uv.cpu().numpy(), z.cpu().numpy())


def default_epsilon(positions) -> float:
    """1% of the bbox diagonal (geometry.py:83-86). Host arithmetic on 6 numbers."""
    if is_torch(positions):
        lo = positions.amin(dim=0).double().cpu().numpy()
        hi = positions.amax(dim=0).double().cpu().numpy()
    else:
        p = np.asarray(positions, dtype=np.float64)
        lo, hi = p.min(axis=0), p.max(axis=0)
    return DEFAULT_EPSILON_FRACTION * float(np.linalg.norm(hi - lo))


def visibility_mask(points, views, epsilon: float):
    """Depth-tested visibility (N, V) bool (geometry.py:89-103)."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(points)
    vs = _views_of(views, with_fmap=False)  # the depth test never reads the feature maps
    if tor and points.dtype == t.float32:
        p, pdt = points.to(dev).contiguous(), _lib.PF_F32
    else:
        p, pdt = to_dev(points, t.float64, dev), _lib.PF_F64
    p = p.reshape(-1, 3)
    n = p.shape[0]
    mask = t.empty((n, vs.nviews), dtype=t.uint8, device=dev)
    _lib.call("pf_visibility_mask", ptr(p), pdt, n, ptr(vs.records_dev), vs.nviews, ptr(vs.depth),
              float(epsilon), ptr(mask), stream_handle())
    return mask.bool() if tor else mask.bool().cpu().numpy()


def estimate_normals(positions, k: int, camera_centers):
    """(normals (N,3) f64, degenerate (N,) bool) from k-NN covariances oriented toward the mean
    camera centre (geometry.py:106-146; pf_estimate_normals: exact grid k-NN, fp64 Jacobi). Positions
    are the cloud's f32 coordinates (bundle.py:158); numpy in -> numpy out, torch -> torch."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(positions)
    p = to_dev(positions, t.float32, dev).reshape(-1, 3)
    n = p.shape[0]
    if k < 3:
        raise ValueError(f"normal estimation needs k >= 3, got {k}")
    if k > n:
        raise ValueError(f"k={k} exceeds point count {n}")
    cc = np.asarray(camera_centers.cpu() if is_torch(camera_centers) else camera_centers, dtype=np.float64)
    centroid = cc.reshape(-1, 3).mean(axis=0)
    normals = t.empty((n, 3), dtype=t.float64, device=dev)
    degen = t.empty(n, dtype=t.uint8, device=dev)
    ws = t.empty(int(_lib.load().pf_normals_workspace_bytes(n)), dtype=t.uint8, device=dev)
    _lib.call("pf_estimate_normals", ptr(p), n, int(k), float(centroid[0]), float(centroid[1]), float(centroid[2]),
              ptr(normals), ptr(degen), ptr(ws), stream_handle())
    if tor:
        return normals, degen.bool()
    return normals.cpu().numpy(), degen.bool().cpu().numpy()
