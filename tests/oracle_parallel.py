"""The CPU oracle over many points in forked worker processes (TEST INFRASTRUCTURE ONLY).

The reference's algorithm is independent per point (visibility, aggregation, grounding), so a
full-size object is checked by splitting its points into chunks, one `oracle.propfield_oracle`
pass per chunk. Voxel codes use the whole object's domain (the GPU indexes the full object's bbox),
so per-point codes of a slice are comparable; the mass needs every point (voxel means).
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_W = {}


def _init():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _chunk(idx):
    from oracle import propfield_oracle as O

    d = _W
    p = d["pts"][idx].astype(np.float64)
    vis = O.visibility_mask(p, d["views"], d["eps"])
    feats, counts = O.aggregate_geometric_features(p, d["views"], vis)
    fhat = O.normalize_rows(feats)
    featured = counts > 0
    k = d["text"].shape[0]
    weights = np.zeros((p.shape[0], k))
    if featured.any():
        sims = O.material_similarity(fhat[featured], d["text"])
        weights[featured] = O.softmax_weights(sims, d["T"])
    props = O.regress_with_weights(weights, d["values"])
    codes, edge = O.voxel_codes(d["pts"][idx], d["grid"], d["lo"], d["hi"])
    return idx, np.packbits(vis, axis=1, bitorder="little"), counts, props, codes, weights.sum(axis=0), edge


def oracle_rows(wl, idx=None, procs: int | None = None) -> dict:
    """Oracle outputs for the points `idx` of workload `wl` (all points when None): packed visibility
    (N, ceil(V/8)) little-endian bits, counts, props (N, P) f64, voxel codes over the FULL object's
    domain, the per-material weight totals of the rows and the voxel edge."""
    pts = wl.points
    idx = np.arange(pts.shape[0]) if idx is None else np.asarray(idx)
    p64 = pts.astype(np.float64)
    _W.update(pts=pts, views=wl.views(f32_maps=True), text=wl.text, values=wl.values, T=wl.cfg.temperature,
              eps=wl.cfg.eps, grid=wl.cfg.grid, lo=p64.min(axis=0), hi=p64.max(axis=0))
    procs = procs or max(1, min(32, len(os.sched_getaffinity(0))))
    chunks = [c for c in np.array_split(idx, procs * 4) if len(c)]
    with mp.get_context("fork").Pool(procs, initializer=_init) as pool:
        parts = pool.map(_chunk, chunks, chunksize=1)
    order = np.argsort(np.concatenate([q[0] for q in parts]), kind="stable")
    cat = lambda j: np.concatenate([q[j] for q in parts])[order]  # noqa: E731
    return {"idx": idx, "vis_bits": cat(1), "counts": cat(2), "props": cat(3), "codes": cat(4),
            "weight_totals": sum(q[5] for q in parts), "edge": parts[0][6]}


def unpack_mask_bits(mask_bits_i32: np.ndarray, nviews: int) -> np.ndarray:
    """GPU bitset words (N, ceil(V/32)) int32 -> (N, V) bool."""
    w = mask_bits_i32.astype(np.int64) & 0xFFFFFFFF
    bits = (w[:, :, None] >> np.arange(32)) & 1
    return bits.reshape(w.shape[0], -1)[:, :nviews].astype(bool)
