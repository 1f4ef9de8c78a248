"""The fused north-star entry: `fuse_and_query`.

One call = project every point into every view, depth-test, bilinear-gather, cross-view mean,
L2-normalise, cosine similarity vs K text embeddings, temperature softmax, property regression,
voxel codes + dense voxel partials and the integrate_mass partial sums — all on the device, with
every intermediate kept in HBM/registers. The per-point results stay on the device; the only
host-visible scalars (mass, partials) are read when the caller asks.

Multi-GPU (point-range sharding): each rank calls `fuse_and_query(..., reduce=False)`
on its point range with the replicated ViewSet and a shared voxel domain, then
`FusedResult.allreduce()` sums the packed partials in ONE NCCL all-reduce, then `finalize()`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import ViewSet, ptr, require_cuda, stream_handle, to_dev, torch
from .errors import BundleStructureError, MaterialError


@dataclass
class QueryTables:
    """Per-object grounding inputs on the device.

    text      (K, D) f32 unit rows (grounding.py:86-93)
    values    (K, P) f32 regressed properties; column `density_col` is density (kg/m^3)
    mid_theta (K,)   f32 mid-range density * thickness (integrate.py:132,146)
    """

    text: object
    values: object
    mid_theta: object
    density_col: int = 0

    @property
    def k(self) -> int:
        return int(self.text.shape[0])

    @property
    def p(self) -> int:
        return int(self.values.shape[1])

    @classmethod
    def build(cls, text, values, mid_theta=None, density_col=0, device=None):
        dev = require_cuda(device)
        t = torch()
        tx = to_dev(text, t.float32, dev)
        vals = to_dev(values, t.float32, dev)
        if vals.dim() == 1:
            vals = vals.reshape(-1, 1)
        if mid_theta is None:
            mid_theta = np.zeros(tx.shape[0], dtype=np.float32)
        mt = to_dev(mid_theta, t.float32, dev).reshape(-1)
        if vals.shape[0] != tx.shape[0] or mt.shape[0] != tx.shape[0]:
            raise BundleStructureError("text, values and mid_theta must have K rows")
        return cls(tx, vals, mt, int(density_col))


class FuseBuffers:
    """Preallocated outputs + workspace for repeated calls (no allocation in the hot loop, CUDA-graph
    capturable). `n` is a CAPACITY: any call with at most n points reuses them (outputs are the
    leading rows); the voxel grid is allocated once and never reallocated or re-zeroed for a new
    point count."""

    def __init__(self, n, views: ViewSet, tables: QueryTables, grid: int, *, features=False,
                 sims=False, weights=False, device=None):
        t = torch()
        dev = views.device if device is None else device
        k, p, nv = tables.k, tables.p, views.nviews
        self.n, self.grid = int(n), int(grid)
        self.capacity = self.n
        nwords = (nv + 31) // 32
        self.counts = t.empty(n, dtype=t.int32, device=dev)
        self.mask_bits = t.empty((n, nwords), dtype=t.int32, device=dev)
        self.props = t.empty((n, p), dtype=t.float32, device=dev)
        self.codes = t.empty(n, dtype=t.int32, device=dev)
        self.grid_partials = t.zeros(2 * grid**3, dtype=t.float32, device=dev)
        # touched-voxel list: on one GPU the mass reduction walks it and re-zeroes those voxels, so
        # the 2 g^3 grid is neither memset nor scanned per object (dense path after an all-reduce)
        self.vox_list = t.full((max(1, 2 * n),), -1, dtype=t.int32, device=dev)
        self.vox_count = t.zeros(1, dtype=t.int32, device=dev)
        self.grid_clean = True
        self.partials = t.zeros(k + 6, dtype=t.float64, device=dev)
        self.mass = t.zeros(2, dtype=t.float64, device=dev)
        self.status = t.zeros(1, dtype=t.int32, device=dev)
        self.lo_hi = t.zeros(6, dtype=t.float64, device=dev)
        self.features = t.empty((n, views.d), dtype=t.float32, device=dev) if features else None
        self.sims = t.empty((n, k), dtype=t.float32, device=dev) if sims else None
        self.weights = t.empty((n, k), dtype=t.float32, device=dev) if weights else None
        args = _make_args(None, n, views, tables, 0.1, 0.01, grid, self, 0)
        ws = int(_lib.load().pf_fuse_workspace_bytes(args))
        self.workspace = t.empty(max(ws, 256), dtype=t.uint8, device=dev)

    def reset(self):
        if not self.grid_clean:
            self.grid_partials.zero_()
            self.grid_clean = True
        self.vox_count.zero_()
        self.partials.zero_()
        self.mass.zero_()
        self.status.zero_()


def _make_args(points, n, views, tables, temperature, eps, grid, b, flags):
    a = _lib.FuseArgs()
    a.points = ptr(points) if points is not None else None
    a.n = int(n)
    a.views = ptr(views.records_dev)
    a.views_host = views.records_host_ptr
    a.nviews = views.nviews
    a.depth = ptr(views.depth)
    a.fmap = ptr(views.fmap)
    a.fmap_dtype = views.fmap_dtype
    a.d = views.d
    a.text = ptr(tables.text)
    a.k = tables.k
    a.values = ptr(tables.values)
    a.p = tables.p
    a.density_col = tables.density_col
    a.mid_theta = ptr(tables.mid_theta)
    a.temperature = float(temperature)
    a.eps = float(eps)
    a.grid = int(grid)
    a.lo_hi = ptr(b.lo_hi)
    a.flags = flags
    a.counts = ptr(b.counts)
    a.mask_bits = ptr(b.mask_bits)
    a.props = ptr(b.props)
    a.codes = ptr(b.codes)
    a.grid_partials = ptr(b.grid_partials)
    a.partials = ptr(b.partials)
    a.status = ptr(b.status)
    a.features = ptr(b.features)
    a.sims = ptr(b.sims)
    a.weights = ptr(b.weights)
    a.workspace = ptr(getattr(b, "workspace", None))
    a.vox_list = ptr(getattr(b, "vox_list", None))
    a.vox_count = ptr(getattr(b, "vox_count", None))
    return a


@dataclass
class FusedResult:
    """Device-resident outputs of one fused call (views into the FuseBuffers)."""

    buffers: FuseBuffers
    nviews: int
    k: int
    n: int = -1  # points of this call (<= buffers.capacity); -1: the whole capacity

    def _rows(self, x):
        return x if (x is None or self.n < 0 or self.n == x.shape[0]) else x[: self.n]

    counts = property(lambda self: self._rows(self.buffers.counts))
    mask_bits = property(lambda self: self._rows(self.buffers.mask_bits))
    props = property(lambda self: self._rows(self.buffers.props))
    codes = property(lambda self: self._rows(self.buffers.codes))
    partials = property(lambda self: self.buffers.partials)
    features = property(lambda self: self._rows(self.buffers.features))
    sims = property(lambda self: self._rows(self.buffers.sims))
    weights = property(lambda self: self._rows(self.buffers.weights))
    lo_hi = property(lambda self: self.buffers.lo_hi)
    mass = property(lambda self: self.buffers.mass)  # (2,) f64 {mass_kg, occupied voxels} after finalize()

    def visibility(self):
        """Unpack the bitset to (N, V) bool (validation helper)."""
        t = torch()
        words = self.mask_bits.to(t.int64) & 0xFFFFFFFF
        bit = t.arange(32, device=words.device, dtype=t.int64)
        bits = ((words[:, :, None] >> bit) & 1).reshape(words.shape[0], -1)
        return bits[:, : self.nviews].bool()

    def allreduce(self, group=None):
        """Sum voxel + integrate partials across ranks (dist.allreduce_partials)."""
        from .dist import allreduce_partials

        allreduce_partials(self.buffers.grid_partials, self.buffers.partials, group)
        self.reduced = True  # the grid now holds other ranks' voxels too: dense finalisation

    def finalize(self):
        """Voxel mass from the (reduced) grid: buffers.mass = {mass_kg, occupied_voxels}."""
        if getattr(self, "finalized", False):  # the sparse pass re-zeroes the grid: run once
            return self
        self.finalized = True
        b = self.buffers
        b.mass.zero_()
        if getattr(self, "reduced", False):
            _lib.call("pf_voxel_mass", ptr(b.grid_partials), b.grid, ptr(b.lo_hi), ptr(b.mass), stream_handle())
            b.grid_clean = False
        else:
            _lib.call("pf_voxel_mass_sparse", ptr(b.grid_partials), b.grid, ptr(b.vox_list), ptr(b.vox_count),
                      int(b.vox_list.numel() // 2), ptr(b.lo_hi), ptr(b.mass), stream_handle())
            b.grid_clean = True
        return self

    def check(self):
        st = int(self.buffers.status.item())
        if st & 1:
            raise MaterialError("NaN similarity passed to kernel regression")
        if st & 2:
            raise MaterialError("non-finite softmax sum (infinite feature or text values)")
        return self

    def mass_kg(self) -> float:
        return float(self.buffers.mass[0].item())

    def host_partials(self) -> dict:
        p = self.partials.cpu().numpy()
        k = self.k
        return {
            "weight_totals": p[:k],
            "pm_sum": p[k],
            "pm_pos": p[k + 1 : k + 4],
            "featured": int(round(p[k + 4])),
            "visible_pairs": int(round(p[k + 5])),
        }


def fuse_and_query(points, views: ViewSet, tables: QueryTables, *, temperature: float = 0.1,
                   epsilon: float = 0.01, grid: int = 64, lo_hi=None, buffers: FuseBuffers | None = None,
                   write_features: bool = False, write_sims: bool = False,
                   write_weights: bool = False, reduce: bool = True, check: bool = False,
                   force_simt: bool = False, prepared: bool = False,
                   reset: bool = True, feature_kernel: bool = False, deterministic: bool = False,
                   depth_ready=None, fmap_ready=None) -> FusedResult:
    """Run the whole path on `points` (N,3) f32 device tensor (numpy is uploaded).

    lo_hi: voxel domain (6,) f64 device tensor; None = this call's bbox (pf_bbox). Multi-GPU
    callers pass the all-reduced global bbox so every rank indexes the same grid.
    reduce=False skips the voxel-mass finalisation (call allreduce() then finalize()).
    bf16 maps run the Gram-formulation tile kernel; write_features (a validation output only the
    feature-product kernel produces) or feature_kernel=True select k_tile_ws instead.
    deterministic=True: run-to-run identical results (stable sort of the points; slower).
    depth_ready / fmap_ready: torch.cuda.Event recorded after the upload of `views`' depth maps /
    feature maps (and `tables.text`), still in flight: the call waits for each only where it is
    first read, so the point sort overlaps the object's remaining uploads (stream.FusePipeline).
    """
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    dev = require_cuda()
    t = torch()
    pts = points if (hasattr(points, "is_cuda") and points.is_cuda and points.dtype == t.float32
                     and points.is_contiguous()) else to_dev(points, t.float32, dev)
    pts = pts.reshape(-1, 3)
    n = pts.shape[0]
    if buffers is None:
        buffers = FuseBuffers(n, views, tables, grid, features=write_features, sims=write_sims,
                              weights=write_weights, device=dev)
    elif reset:
        buffers.reset()
    if n > buffers.capacity or buffers.grid != grid:
        raise BundleStructureError(f"buffers hold {buffers.capacity} points on a {buffers.grid}^3 grid; "
                                   f"this call has {n} points on {grid}^3")
    st = stream_handle()
    if lo_hi is None:
        if n == 0:
            buffers.lo_hi.zero_()
        else:
            _lib.call("pf_bbox", ptr(pts), n, ptr(buffers.lo_hi), st)
    else:
        buffers.lo_hi.copy_(to_dev(lo_hi, t.float64, dev).reshape(6))
    flags = 0
    if write_features:
        flags |= _lib.PF_FUSE_WRITE_FEATURES
    if write_sims:
        flags |= _lib.PF_FUSE_WRITE_SIMS
    if write_weights:
        flags |= _lib.PF_FUSE_WRITE_WEIGHTS
    if force_simt:
        flags |= _lib.PF_FUSE_FORCE_SIMT
    if prepared:
        flags |= _lib.PF_FUSE_PREPARED
    if feature_kernel:
        flags |= _lib.PF_FUSE_FEATURE_KERNEL
    if deterministic:
        flags |= _lib.PF_FUSE_DETERMINISTIC
    args = _make_args(pts, n, views, tables, temperature, epsilon, grid, buffers, flags)
    args.depth_ready = depth_ready.cuda_event if depth_ready is not None else None
    args.fmap_ready = fmap_ready.cuda_event if fmap_ready is not None else None
    _lib.call("pf_fuse_query", args, st)
    res = FusedResult(buffers, views.nviews, tables.k, n)
    # the grid now holds this call's voxels until finalize() re-zeroes the touched ones (sparse) or
    # marks it for a full reset (dense): an un-finalised grid must be zeroed by the next reset()
    buffers.grid_clean = False
    if reduce:
        res.finalize()
    if check:
        res.check()
    return res


def fuse_prepare(views: ViewSet, tables: QueryTables, buffers: FuseBuffers) -> None:
    """Per-object tables (G = fmap @ text^T) into `buffers.workspace` (pf_fuse_prepare); pass
    `prepared=True` to the following fuse_and_query calls on the same object."""
    args = _make_args(None, buffers.n, views, tables, 0.1, 0.01, buffers.grid, buffers, 0)
    _lib.call("pf_fuse_prepare", args, stream_handle())
