"""Geometric feature lifting (reference fusion.py:65-93) on the GPU.

`aggregate_geometric_features(positions, views, visibility)` keeps the reference signature and
returns a `SemanticPointCloud` whose `features` are bit-identical to the reference's float64
means: per channel the device accumulates in fp64 over visible views in view order, exactly like
`accum[rows] += sampled` followed by one division (fusion.py:75-90).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import cached_view_set, is_torch, ptr, require_cuda, stream_handle, to_dev, torch
from .errors import BundleStructureError
from .types import SemanticPointCloud


def aggregate_geometric_features(positions, views, visibility) -> SemanticPointCloud:
    dev = require_cuda()
    t = torch()
    tor = is_torch(positions)
    vs = cached_view_set(views)  # uploaded once per view list (device.cached_view_set)
    if tor and positions.dtype == t.float32:
        p, pdt = positions.to(dev).contiguous(), _lib.PF_F32
    else:
        p, pdt = to_dev(positions, t.float64, dev), _lib.PF_F64
    p = p.reshape(-1, 3)
    n = p.shape[0]
    vis = to_dev(visibility, t.uint8, dev)
    if tuple(vis.shape) != (n, vs.nviews):
        raise BundleStructureError(
            f"visibility must be ({n}, {vs.nviews}), got {tuple(vis.shape)}"
        )
    feats = t.empty((n, vs.d), dtype=t.float64, device=dev)
    counts = t.empty(n, dtype=t.int64, device=dev)
    _lib.call("pf_aggregate_features", ptr(p), pdt, n, ptr(vs.records_dev), vs.nviews,
              ptr(vs.fmap), vs.fmap_dtype, vs.d, ptr(vis), ptr(feats), ptr(counts),
              stream_handle())
    if tor:
        return SemanticPointCloud(positions=p.double(), features=feats, visible_counts=counts,
                                  visibility=vis.bool())
    return SemanticPointCloud(
        positions=np.atleast_2d(np.asarray(positions, dtype=np.float64)),
        features=feats.cpu().numpy(),
        visible_counts=counts.cpu().numpy(),
        visibility=np.asarray(visibility),
    )
