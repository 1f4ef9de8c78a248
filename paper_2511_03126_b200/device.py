"""Device plumbing: streams, tensor conversion and the packed per-view layout in HBM.

HBM layout of a view set (one per object; replicated per GPU under point sharding):

* `records`  — V x pf_view_t (160 B each): fp64 R, t, intrinsics + element offsets + sizes;
* `depth`    — all (H, W) f32 z-depth maps back to back (bundle.py:101-116 dtype);
* `fmap`     — all (Hf, Wf, D) channel-last maps back to back, f32 or bf16 (bf16-feature mode:
               SURVEY §8a-13). Channel-last keeps each cell's D channels contiguous so a warp's
               16-byte lane loads of one tap are one coalesced 512-byte transaction.

PyTorch provides the allocator and the current stream; everything computed runs in the native
library.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import BundleStructureError, CudaError
from .types import feature_dtype_of


def torch():
    import torch as _t

    return _t


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise CudaError("no CUDA device: the propfield B200 path has no CPU fallback")
    _lib.load()
    return t.device("cuda", t.cuda.current_device() if device is None else t.device(device).index)


def stream_handle() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def to_dev(x, dtype, device):
    """numpy / torch -> contiguous tensor of `dtype` on `device` (H2D copy when needed)."""
    t = torch()
    if isinstance(x, t.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(x)
    return t.from_numpy(arr).to(device=device, dtype=dtype, non_blocking=False).contiguous()


def fmap_to_dev(fm, kind: str, device):
    """A feature map as a device tensor: float32 or bfloat16 (numpy uint16 = bf16 bits)."""
    t = torch()
    if isinstance(fm, t.Tensor):
        want = t.bfloat16 if kind == "bf16" else t.float32
        return fm.to(device=device, dtype=want).contiguous()
    arr = np.ascontiguousarray(fm)
    if kind == "bf16":
        if arr.dtype != np.uint16:
            raise BundleStructureError("bf16 feature maps on the host must be uint16 bit patterns")
        return t.from_numpy(arr.view(np.int16)).to(device).view(t.bfloat16).contiguous()
    return t.from_numpy(arr.astype(np.float32, copy=False)).to(device).contiguous()


class ViewSet:
    """V views packed for the device. Build once per object and reuse across calls."""

    def __init__(self, records: np.ndarray, depth, fmap, fmap_kind: str, d: int, device):
        t = torch()
        self.records = records
        self.records_dev = t.from_numpy(records.view(np.uint8).copy()).to(device)
        self.depth = depth
        self.fmap = fmap
        self.fmap_kind = fmap_kind
        self.fmap_dtype = _lib.PF_BF16 if fmap_kind == "bf16" else _lib.PF_F32
        self.d = int(d)
        self.device = device

    @property
    def nviews(self) -> int:
        return int(self.records.shape[0])

    @property
    def records_host_ptr(self) -> int:
        return self.records.ctypes.data

    def record(self, j: int) -> np.ndarray:
        return self.records[j : j + 1]

    @classmethod
    def from_views(cls, views, device=None, fmap_kind: str | None = None, with_fmap: bool = True) -> "ViewSet":
        """Pack reference-style view records (bundle.py:93-139 attribute names). with_fmap=False
        uploads records + depth only (the records still carry the maps' offsets and sizes, read from
        their shapes); `attach_fmaps` adds the maps later."""
        dev = require_cuda(device)
        t = torch()
        views = list(views)
        if not views:
            raise BundleStructureError("at least one view is required")
        dims = {int(v.feature_map.shape[2]) for v in views}
        if len(dims) != 1:
            raise BundleStructureError(f"feature dimension differs across views: {sorted(dims)}")
        d = dims.pop()
        kinds = {getattr(v, "feature_dtype", None) or feature_dtype_of(v.feature_map) for v in views}
        kinds.discard("auto")
        if not kinds:
            kinds = {feature_dtype_of(v.feature_map) for v in views}
        kind = fmap_kind or ("bf16" if kinds == {"bf16"} else "f32")
        rec = np.zeros(len(views), dtype=_lib.VIEW_DTYPE)
        depth_parts, fmap_parts = [], []
        doff = foff = 0
        for j, v in enumerate(views):
            cam, intr = v.camera, v.intrinsics
            dm = np.asarray(v.depth, dtype=np.float32)
            h, w = dm.shape
            hf, wf = int(v.feature_map.shape[0]), int(v.feature_map.shape[1])
            rec[j]["R"] = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
            rec[j]["t"] = np.asarray(cam.translation, dtype=np.float64)
            rec[j]["fx"], rec[j]["fy"] = float(intr.fx), float(intr.fy)
            rec[j]["cx"], rec[j]["cy"] = float(intr.cx), float(intr.cy)
            rec[j]["depth_offset"], rec[j]["fmap_offset"] = doff, foff
            rec[j]["H"], rec[j]["W"], rec[j]["Hf"], rec[j]["Wf"] = h, w, hf, wf
            depth_parts.append(t.from_numpy(np.ascontiguousarray(dm)).reshape(-1))
            doff += h * w
            foff += hf * wf * d
        depth = t.cat(depth_parts).to(dev)
        vs = cls(rec, depth, None, kind, d, dev)
        if with_fmap:
            vs.attach_fmaps(views)
        return vs

    def attach_fmaps(self, views) -> "ViewSet":
        """Upload the views' feature maps into the packed channel-last block (no-op if present)."""
        if self.fmap is not None:
            return self
        t = torch()
        parts = []
        for v in views:
            vk = getattr(v, "feature_dtype", None) or feature_dtype_of(v.feature_map)
            fm = fmap_to_dev(v.feature_map, vk if vk in ("f32", "bf16") else "f32", self.device)
            parts.append(fm.to(t.bfloat16 if self.fmap_kind == "bf16" else t.float32).reshape(-1))
        self.fmap = t.cat(parts).contiguous()
        return self

    @classmethod
    def from_tensors(cls, R, tvec, intr, depth, fmap, device=None) -> "ViewSet":
        """Uniform-size views from stacked arrays: R (V,3,3) f64, t (V,3), intr (V,4)
        [fx,fy,cx,cy], depth (V,H,W) f32 tensor, fmap (V,Hf,Wf,D) f32|bf16 tensor."""
        dev = require_cuda(device)
        t = torch()
        R = np.asarray(R, dtype=np.float64)
        tvec = np.asarray(tvec, dtype=np.float64)
        intr = np.asarray(intr, dtype=np.float64)
        nv, h, w = (int(s) for s in depth.shape)
        _, hf, wf, d = (int(s) for s in fmap.shape)
        rec = np.zeros(nv, dtype=_lib.VIEW_DTYPE)
        rec["R"] = R.reshape(nv, 9)
        rec["t"] = tvec
        rec["fx"], rec["fy"], rec["cx"], rec["cy"] = intr[:, 0], intr[:, 1], intr[:, 2], intr[:, 3]
        rec["depth_offset"] = np.arange(nv, dtype=np.int64) * h * w
        rec["fmap_offset"] = np.arange(nv, dtype=np.int64) * hf * wf * d
        rec["H"], rec["W"], rec["Hf"], rec["Wf"] = h, w, hf, wf
        kind = "bf16" if fmap.dtype == t.bfloat16 else "f32"
        return cls(
            rec,
            depth.to(dev, t.float32).contiguous().reshape(-1),
            fmap.to(dev).contiguous().reshape(-1),
            kind,
            d,
            dev,
        )


# ---- per-object view cache of the drop-in op API ------------------------------------------------
# The reference's pipeline calls visibility_mask and then aggregate_geometric_features on the same
# view list (pipeline.py:225-232). Both take reference-style views, so without a cache each call
# re-packs and re-uploads every depth map and feature map. The cache keys on the identity of the
# view objects and of their depth / feature arrays and keeps strong references to them (an id cannot
# be recycled while its entry lives), so rebinding `view.depth` or `view.feature_map` is a miss.
# In-place writes into a cached array are NOT detected: call clear_view_cache() after mutating one.
_VIEW_CACHE: "dict" = {}
_VIEW_CACHE_ORDER: list = []
VIEW_CACHE_SIZE = 2  # objects (a C5 object's views are 243 MB of HBM)


def _view_key(views, device) -> tuple:
    return (str(device),) + tuple((id(v), id(v.depth), id(v.feature_map)) for v in views)


def clear_view_cache() -> None:
    _VIEW_CACHE.clear()
    _VIEW_CACHE_ORDER.clear()


def cached_view_set(views, with_fmap: bool = True, device=None) -> ViewSet:
    """ViewSet of a reference-style view list, packed and uploaded once per list (see above);
    visibility-only callers ask for with_fmap=False and never upload the feature maps."""
    if isinstance(views, ViewSet):
        return views
    dev = require_cuda(device)
    views = list(views)
    key = _view_key(views, dev)
    hit = _VIEW_CACHE.get(key)
    if hit is None:
        vs = ViewSet.from_views(views, dev, with_fmap=with_fmap)
        # strong refs: the views and their arrays outlive the entry, so the ids stay theirs
        _VIEW_CACHE[key] = (vs, views, [(v.depth, v.feature_map) for v in views])
        _VIEW_CACHE_ORDER.append(key)
        while len(_VIEW_CACHE_ORDER) > VIEW_CACHE_SIZE:
            _VIEW_CACHE.pop(_VIEW_CACHE_ORDER.pop(0), None)
    else:
        vs = hit[0]
        _VIEW_CACHE_ORDER.remove(key)
        _VIEW_CACHE_ORDER.append(key)
    if with_fmap:
        vs.attach_fmaps(views)
    return vs
