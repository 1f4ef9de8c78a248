"""Material grounding math (reference grounding.py:158-202) on the GPU, fp64.

Same names, signatures, return shapes and errors as the reference:
`material_similarity` (plain dot of unit vectors), `softmax_weights` (T <= 0 -> ValueError, NaN ->
MaterialError), `kernel_regress`, `regress_with_weights` ((K,) or (K,2) values).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import is_torch, ptr, require_cuda, stream_handle, to_dev, torch
from .errors import BundleStructureError, MaterialError


def _as2d(x, dev):
    t = torch()
    a = to_dev(x, t.float64, dev)
    return a.reshape(1, -1) if a.dim() == 1 else a


def material_similarity(features, text_embeddings):
    """(S, K) = features (S, D) @ text (K, D)^T (grounding.py:158-165)."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(features) or is_torch(text_embeddings)
    f = _as2d(features, dev)
    tx = _as2d(text_embeddings, dev)
    if f.shape[1] != tx.shape[1]:
        raise BundleStructureError(f"feature dim {f.shape[1]} != text dim {tx.shape[1]}")
    s, d, k = f.shape[0], f.shape[1], tx.shape[0]
    out = t.empty((s, k), dtype=t.float64, device=dev)
    _lib.call("pf_material_similarity", ptr(f), s, d, ptr(tx), k, ptr(out), stream_handle())
    return out if tor else out.cpu().numpy()


def softmax_weights(similarities, temperature: float):
    """Temperature softmax over materials, max-subtracted (grounding.py:168-178)."""
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    dev = require_cuda()
    t = torch()
    tor = is_torch(similarities)
    s = _as2d(similarities, dev)
    n, k = s.shape
    w = t.empty((n, k), dtype=t.float64, device=dev)
    flag = t.zeros(1, dtype=t.int32, device=dev)
    _lib.call("pf_softmax_weights", ptr(s), n, k, float(temperature), None, ptr(w), ptr(flag),
              stream_handle())
    if int(flag.item()):
        raise MaterialError("NaN similarity passed to kernel regression")
    return w if tor else w.cpu().numpy()


def regress_with_weights(weights, values):
    """Convex combination (S,K) @ (K,) or (K,P) (grounding.py:198-202)."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(weights) or is_torch(values)
    w = _as2d(weights, dev)
    y = to_dev(values, t.float64, dev)
    vec = y.dim() == 1
    y2 = y.reshape(-1, 1) if vec else y
    if y2.shape[0] != w.shape[1]:
        raise BundleStructureError(f"values have {y2.shape[0]} rows, weights {w.shape[1]} columns")
    s, k, p = w.shape[0], w.shape[1], y2.shape[1]
    out = t.empty((s, p), dtype=t.float64, device=dev)
    _lib.call("pf_regress_with_weights", ptr(w), s, k, ptr(y2.contiguous()), p, ptr(out),
              stream_handle())
    out = out.reshape(-1) if vec else out
    return out if tor else out.cpu().numpy()


def kernel_regress(similarities, values, temperature: float):
    """regress_with_weights(softmax_weights(s, T), values) (grounding.py:181-195)."""
    return regress_with_weights(softmax_weights(similarities, temperature), values)
