"""View scoring of the anchor set on the GPU: view_select.score_views / rank_views
(view_select.py:51-124), same signatures, return types and tie-breaking (pf_score_views)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import ViewSet, cached_view_set, ptr, require_cuda, stream_handle, to_dev, torch


@dataclass
class ViewScore:
    """view_select.py:21-29."""

    point_index: int
    view_index: int
    z: float
    s_dist: float
    s_angle: float
    s_total: float
    pixel: tuple


def _run(source, views, visibility, k):
    if source.normals is None:
        raise ValueError("source set has no normals; run normal estimation first")
    dev = require_cuda()
    t = torch()
    vs = cached_view_set(views, with_fmap=False)  # cameras only
    pos = to_dev(source.positions, t.float64, dev).reshape(-1, 3)
    nrm = to_dev(source.normals, t.float64, dev).reshape(-1, 3)
    s, nv = pos.shape[0], vs.nviews
    vis = to_dev(np.asarray(visibility, dtype=np.uint8) if not hasattr(visibility, "cpu") else visibility.to(t.uint8),
                 t.uint8, dev).reshape(s, nv)
    out = {n: t.empty((s, nv), dtype=t.float64, device=dev) for n in ("s_total", "s_angle", "z")}
    pix = t.empty((s, nv, 2), dtype=t.float64, device=dev)
    ranked = t.empty((s, max(1, k)), dtype=t.int32, device=dev)
    _lib.call("pf_score_views", ptr(pos), ptr(nrm), s, ptr(vs.records_dev), nv, ptr(vis), ptr(out["s_total"]),
              ptr(out["s_angle"]), ptr(out["z"]), ptr(pix), int(k), ptr(ranked), stream_handle())
    return out, pix, ranked


def score_views(source, views, visibility):
    """(s_total, s_angle, z, pixels) numpy arrays (view_select.py:51-80)."""
    out, pix, _ = _run(source, views, visibility, 1)
    return out["s_total"].cpu().numpy(), out["s_angle"].cpu().numpy(), out["z"].cpu().numpy(), pix.cpu().numpy()


def rank_views(source, views, visibility, k: int):
    """Top-k visible views per anchor, ties toward the lower view index (view_select.py:83-124);
    anchors visible nowhere get [] and source.flags["zero_visible"]."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    out, pix, ranked = _run(source, views, visibility, k)
    st, sa, z, px, rk = (out["s_total"].cpu().numpy(), out["s_angle"].cpu().numpy(), out["z"].cpu().numpy(),
                         pix.cpu().numpy(), ranked.cpu().numpy())
    rankings, zero = [], np.zeros(rk.shape[0], dtype=np.bool_)
    for i in range(rk.shape[0]):
        entries = []
        for j in rk[i]:
            if j < 0:
                break
            zz = float(z[i, j])
            entries.append(ViewScore(point_index=i, view_index=int(j), z=zz, s_dist=float(1.0 / (1.0 + zz)),
                                     s_angle=float(sa[i, j]), s_total=float(st[i, j]),
                                     pixel=(float(px[i, j, 0]), float(px[i, j, 1]))))
        zero[i] = not entries
        rankings.append(entries)
    if not hasattr(source, "flags") or source.flags is None:
        source.flags = {}
    source.flags["zero_visible"] = zero
    return rankings
