"""The reference's kernel registry (`propfield.kernels`, kernels/__init__.py:1-101), B200 edition.

Same three hot-path operator names and signatures as the reference's numba/numpy twins
(numpy_impl.py:14-77, numba_impl.py:15-89), executed by fp64 CUDA kernels that keep the
reference's operation order, so results are bit-identical to the numpy build (the reference's own
cross-backend test uses rtol=atol=0, tests/test_kernels.py:19-57).

There is exactly one backend, "cuda": `set_backend` accepts only that name (no multi-backend
dispatch, no CPU fallback). numpy inputs are copied to the GPU and results copied back; torch
CUDA tensors stay on the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import is_torch, ptr, require_cuda, stream_handle, to_dev, torch
from .errors import BundleStructureError
from .types import feature_dtype_of

_KERNEL_NAMES = ["visible_in_view", "bilinear_gather", "accumulate_features"]
_BACKEND = "cuda"


def set_backend(name: str) -> None:
    """Select the kernel backend; only "cuda" exists (kernels/__init__.py:53-64)."""
    if name != _BACKEND:
        raise ValueError(f"unknown kernel backend {name!r} (this build has only 'cuda')")


def active_backend() -> str:
    return _BACKEND


def available_backends() -> list:
    return [_BACKEND]


def get_impl(name: str | None = None):
    if name not in (None, _BACKEND):
        raise ValueError(f"unknown kernel backend {name!r}")
    import sys

    return sys.modules[__name__]


def warmup() -> None:
    """Load the library and create the CUDA context (kernels/__init__.py:88-91)."""
    require_cuda()
    torch().cuda.synchronize()


def _ret(arr, like_torch: bool):
    return arr if like_torch else arr.cpu().numpy()


def _fmap_dev(fmap, dev):
    t = torch()
    kind = feature_dtype_of(fmap)
    if is_torch(fmap):
        f = fmap.to(dev).contiguous()
        if f.dtype not in (t.float32, t.bfloat16):
            f = f.to(t.float32)
    elif kind == "bf16":
        f = t.from_numpy(np.ascontiguousarray(fmap).view(np.int16)).to(dev).view(t.bfloat16)
    else:
        f = to_dev(fmap, t.float32, dev)
    code = _lib.PF_BF16 if f.dtype == t.bfloat16 else _lib.PF_F32
    if f.dim() != 3:
        raise BundleStructureError(f"feature map must be (Hf, Wf, D), got {tuple(f.shape)}")
    return f, code


def visible_in_view(u, v, z, depth_map, eps):
    """Depth-test projected points against one view's depth map (numpy_impl.py:14-40)."""
    dev = require_cuda()
    t = torch()
    tor = any(is_torch(x) for x in (u, v, z, depth_map))
    ud, vd, zd = (to_dev(x, t.float64, dev).reshape(-1) for x in (u, v, z))
    dm = to_dev(depth_map, t.float32, dev)
    if dm.dim() != 2:
        raise BundleStructureError(f"depth map must be (H, W), got {tuple(dm.shape)}")
    n = ud.shape[0]
    out = t.empty(n, dtype=t.uint8, device=dev)
    _lib.call("pf_visible_in_view", ptr(ud), ptr(vd), ptr(zd), n, ptr(dm), dm.shape[0],
              dm.shape[1], float(eps), ptr(out), stream_handle())
    return _ret(out.bool(), tor)


def bilinear_gather(fmap, fu, fv):
    """Border-clamped bilinear samples (M, D) float64 (numpy_impl.py:43-66)."""
    dev = require_cuda()
    t = torch()
    tor = any(is_torch(x) for x in (fmap, fu, fv))
    f, code = _fmap_dev(fmap, dev)
    fud, fvd = (to_dev(x, t.float64, dev).reshape(-1) for x in (fu, fv))
    hf, wf, d = (int(s) for s in f.shape)
    m = fud.shape[0]
    out = t.empty((m, d), dtype=t.float64, device=dev)
    _lib.call("pf_bilinear_gather", ptr(f), code, hf, wf, d, ptr(fud), ptr(fvd), m, ptr(out),
              stream_handle())
    return _ret(out, tor)


def accumulate_features(fmap, fu, fv, rows, accum, counts):
    """accum[rows] += bilinear samples; counts[rows] += 1, IN PLACE (numpy_impl.py:69-77).

    `accum` (N, D) float64 and `counts` (N,) int64 are the caller's buffers: torch CUDA tensors are
    updated on the device; numpy arrays are round-tripped through the GPU and overwritten."""
    dev = require_cuda()
    t = torch()
    f, code = _fmap_dev(fmap, dev)
    fud, fvd = (to_dev(x, t.float64, dev).reshape(-1) for x in (fu, fv))
    rws = to_dev(rows, t.int64, dev).reshape(-1)
    hf, wf, d = (int(s) for s in f.shape)
    m = fud.shape[0]
    inplace = is_torch(accum) and accum.is_cuda and accum.dtype == t.float64 and accum.is_contiguous()
    acc = accum if inplace else to_dev(accum, t.float64, dev)
    cinplace = is_torch(counts) and counts.is_cuda and counts.dtype == t.int64 and counts.is_contiguous()
    cnt = counts if cinplace else to_dev(counts, t.int64, dev)
    if acc.dim() != 2 or acc.shape[1] != d:
        raise BundleStructureError(f"accumulator must be (N, {d}), got {tuple(acc.shape)}")
    _lib.call("pf_accumulate_features", ptr(f), code, hf, wf, d, ptr(fud), ptr(fvd), ptr(rws), m,
              ptr(acc), ptr(cnt), stream_handle())
    if not inplace:
        if is_torch(accum):
            accum.copy_(acc)
        else:
            accum[...] = acc.cpu().numpy()
    if not cinplace:
        if is_torch(counts):
            counts.copy_(cnt)
        else:
            counts[...] = cnt.cpu().numpy()
