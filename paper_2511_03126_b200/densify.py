"""Densification on the GPU: reference densify.py:36-160, same names and semantics.

* `dino_knn_interpolate(query_features, source_features, source_probs, k)` — cosine k-NN in feature
  space + clamped, renormalised weights (pf_dino_knn_interpolate, fp64). The neighbour order is the
  reference's (similarity desc, index asc). Exact ties AT the k-th place are resolved by the lower
  index; the reference leaves those to np.argpartition (implementation-defined).
* `densify_field(semantic_cloud, source, dictionary, k, normals=None) -> PropertyField` — featured
  points interpolate, featureless ones copy their nearest featured neighbour (pf_nearest_index),
  properties regress on the dictionary's [lo, hi] tables (pf_regress_with_weights).
numpy in -> numpy out; torch CUDA in -> torch out. Queries are processed in chunks so the (Q, S)
similarity workspace stays bounded.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import is_torch, ptr, require_cuda, stream_handle, to_dev, torch
from .errors import BundleStructureError, MaterialError
from .grounding import regress_with_weights
from .types import PropertyField

QUERY_CHUNK = 1 << 20


def _2d(x, dev):
    t = torch()
    a = to_dev(x, t.float64, dev)
    return a.reshape(1, -1) if a.dim() == 1 else a


def dino_knn_interpolate(query_features, source_features, source_probs, k: int):
    """(Q, M) interpolated probability rows (densify.py:36-86)."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(query_features)
    q = _2d(query_features, dev)
    s = _2d(source_features, dev)
    p = _2d(source_probs, dev)
    if k < 1 or k > s.shape[0]:
        raise ValueError(f"k={k} outside 1..{s.shape[0]}")
    if q.shape[1] != s.shape[1]:
        raise BundleStructureError(f"query dim {q.shape[1]} != source dim {s.shape[1]}")
    if p.shape[0] != s.shape[0]:
        raise BundleStructureError(f"{p.shape[0]} probability rows for {s.shape[0]} sources")
    nq, ns, d, m = q.shape[0], s.shape[0], q.shape[1], p.shape[1]
    out = t.empty((nq, m), dtype=t.float64, device=dev)
    chunk = max(1, min(QUERY_CHUNK, nq))
    ws = t.empty(int(_lib.load().pf_dino_knn_workspace_bytes(chunk, ns, d)), dtype=t.uint8, device=dev)
    for a in range(0, nq, chunk):
        b = min(nq, a + chunk)
        try:
            _lib.call("pf_dino_knn_interpolate", ptr(q[a:b]), b - a, ptr(s), ns, d, ptr(p), m, int(k), ptr(out[a:b]),
                      None, ptr(ws), stream_handle())
        except MaterialError as e:
            if a == 0:
                raise
            # re-number the chunk-local indices in the message
            msg = str(e)
            lo, hi = msg.index("[") + 1, msg.index("]")
            nums = [int(x) + a for x in msg[lo:hi].split(",") if x.strip()]
            raise MaterialError(f"query features missing for indices {nums}") from None
    return out if tor else out.cpu().numpy()


BRUTE_FORCE_MAX = 1 << 24  # query x point pairs below which the brute-force kernel is used


def nearest_index(queries, points, grid: bool | None = None):
    """Index of the nearest point (fp64, lowest index on ties) for every query (cKDTree k=1):
    brute force for small sets, the exact grid search otherwise."""
    dev = require_cuda()
    t = torch()
    qq = to_dev(queries, t.float64, dev).reshape(-1, 3)
    pp = to_dev(points, t.float64, dev).reshape(-1, 3)
    idx = t.empty(qq.shape[0], dtype=t.int64, device=dev)
    nq, np_ = qq.shape[0], pp.shape[0]
    if grid is None:
        grid = nq * np_ > BRUTE_FORCE_MAX
    if grid and np_ > 0:
        ws = t.empty(int(_lib.load().pf_nearest_workspace_bytes(np_)), dtype=t.uint8, device=dev)
        _lib.call("pf_nearest_index_grid", ptr(qq), nq, ptr(pp), np_, ptr(idx), ptr(ws), stream_handle())
    else:
        _lib.call("pf_nearest_index", ptr(qq), nq, ptr(pp), np_, ptr(idx), stream_handle())
    return idx


def densify_field(semantic_cloud, source, dictionary, k: int, normals=None) -> PropertyField:
    """densify.py:110-160 on the device; returns a PropertyField with numpy arrays."""
    if source.probabilities is None:
        raise ValueError("source set has no material probabilities; ground it first")
    dev = require_cuda()
    t = torch()
    n = len(semantic_cloud)
    k = min(k, len(source))
    feats = to_dev(semantic_cloud.features, t.float64, dev)
    counts = to_dev(semantic_cloud.visible_counts, t.int64, dev)
    featureless = (counts == 0) | (t.linalg.vector_norm(feats, dim=1) == 0)
    probs = t.zeros((n, len(dictionary)), dtype=t.float64, device=dev)
    featured = t.nonzero(~featureless).reshape(-1)
    if featured.numel():
        probs[featured] = dino_knn_interpolate(feats[featured], to_dev(source.features, t.float64, dev),
                                               to_dev(source.probabilities, t.float64, dev), k)
    orphan = t.nonzero(featureless).reshape(-1)
    if orphan.numel():
        if featured.numel() == 0:
            raise MaterialError("no point in the cloud has a geometric feature")
        pos = to_dev(semantic_cloud.positions, t.float64, dev)
        nn = nearest_index(pos[orphan], pos[featured])
        probs[orphan] = probs[featured[nn]]
    properties = {}
    for prop in dictionary.property_names:
        lo_hi = dictionary.property_values(prop)
        if np.all(lo_hi[:, 0] == lo_hi[:, 1]):
            properties[prop] = regress_with_weights(probs, lo_hi[:, 0]).cpu().numpy()
        else:
            properties[prop] = regress_with_weights(probs, lo_hi).cpu().numpy()
    pr = probs.cpu().numpy()
    return PropertyField(positions=semantic_cloud.positions, probabilities=pr, dominant=np.argmax(pr, axis=1),
                         properties=properties, material_names=dictionary.names, normals=normals,
                         flags={"featureless": featureless.cpu().numpy()})
