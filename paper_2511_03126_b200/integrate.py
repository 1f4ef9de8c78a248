"""Mass integration on the GPU: the reference's integrate_mass (integrate.py:98-167) and the
BASELINE voxel-grid mass.

The data-parallel part of integrate_mass — weight_totals_k = sum_i w_ik, the point masses
pm_i = w_i . (mid * theta) and their position moments — runs on the device (inside the fused kernel
on the fused path, or from a probability matrix here: pf_integrate_partials). The characteristic
length L (integrate.py:72-95, the k=8 nearest-neighbour area estimate) runs on the
device too (pf_knn_kth_distance: exact k-NN over a hashed grid). What remains is O(K) host
arithmetic in the reference's order (integrate.py:128-155).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import is_torch, ptr, require_cuda, stream_handle, to_dev, torch
from .types import IntegrationConfig, ObjectEstimate

AREA_KNN = 8  # integrate.py:19


def adaptive_voxel_side(length: float, scale_factor: float, n_points: int) -> float:
    """sqrt((L * scale_factor)^2 / N) (integrate.py:63-69)."""
    if length < 0:
        raise ValueError(f"characteristic length must be >= 0, got {length}")
    if n_points < 1:
        raise ValueError(f"point count must be >= 1, got {n_points}")
    return float(np.sqrt((length * scale_factor) ** 2 / n_points))


def estimate_from_partials(weight_totals, pm_sum, pm_pos, n, dictionary, config: IntegrationConfig,
                           length: float, mean_position=None) -> ObjectEstimate:
    """Finish integrate_mass from its partial sums, in the reference's operation order
    (integrate.py:124-167). `pm_*` exclude the lam * b^2 factor, which is applied here."""
    if n == 0:
        return ObjectEstimate(0.0, (0.0, 0.0), np.zeros(3), {nm: 0.0 for nm in dictionary.names},
                              0.0, 0.0, 0, config.lam, config.scale_factor)
    density = dictionary.property_values("density")
    theta = dictionary.thicknesses()
    b = adaptive_voxel_side(length, config.scale_factor, n)
    cell_area = b * b
    mid_density = (density[:, 0] + density[:, 1]) / 2.0
    per_material, mass_total, mass_lo, mass_hi = {}, 0.0, 0.0, 0.0
    for idx, name in enumerate(dictionary.names):
        contrib = config.lam * cell_area * theta[idx] * float(weight_totals[idx])
        per_material[name] = contrib * mid_density[idx]
        mass_total += per_material[name]
        mass_lo += contrib * density[idx, 0]
        mass_hi += contrib * density[idx, 1]
    total = config.lam * cell_area * pm_sum
    if total > 0:
        com = np.asarray(pm_pos, dtype=np.float64) / pm_sum
    else:
        com = np.asarray(mean_position if mean_position is not None else np.zeros(3), np.float64)
    return ObjectEstimate(float(mass_total), (float(mass_lo), float(mass_hi)), com, per_material, b,
                          float(length), int(n), config.lam, config.scale_factor)


def characteristic_length(positions, k: int = AREA_KNN) -> float:
    """integrate.characteristic_length (integrate.py:72-95): sqrt(pi / k * sum_i d_k(i)^2) with d_k
    the distance to the (k+1)-th nearest point, self included; the longest bbox axis below 4 points."""
    dev = require_cuda()
    t = torch()
    p = to_dev(positions, t.float32, dev).reshape(-1, 3)
    n = int(p.shape[0])
    if n == 0:
        return 0.0
    if n < 4:
        q = p.double().cpu().numpy()
        return float((q.max(axis=0) - q.min(axis=0)).max())
    k_eff = min(int(k), n - 1)
    lib = _lib.load()
    ws = t.empty(int(lib.pf_knn_workspace_bytes(n)), dtype=t.uint8, device=dev)
    out = t.zeros(1, dtype=t.float64, device=dev)
    _lib.call("pf_knn_kth_distance", ptr(p), n, k_eff, ptr(out), None, ptr(ws), stream_handle())
    return float(np.sqrt(np.pi / k_eff * float(out.item())))


def integrate_mass(fld, dictionary, config: IntegrationConfig) -> ObjectEstimate:
    """integrate.integrate_mass (integrate.py:98-167) on the device: characteristic length by
    device k-NN, weight totals / point-mass moments by pf_integrate_partials, then the reference's
    O(K) arithmetic (estimate_from_partials)."""
    n = len(fld)
    if n == 0:
        return estimate_from_partials(np.zeros(0), 0.0, np.zeros(3), 0, dictionary, config, 0.0)
    dev = require_cuda()
    t = torch()
    density = dictionary.property_values("density")
    theta = np.asarray(dictionary.thicknesses(), np.float64)
    mid = (density[:, 0] + density[:, 1]) / 2.0
    k = int(theta.shape[0])
    w = to_dev(fld.probabilities, t.float64, dev).reshape(n, k)
    pos = to_dev(fld.positions, t.float32, dev).reshape(n, 3)
    nrm = None if fld.normals is None else to_dev(fld.normals, t.float32, dev).reshape(n, 3)
    mt = to_dev(mid * theta, t.float64, dev)
    th = to_dev(theta, t.float64, dev)
    out = t.zeros(k + 4, dtype=t.float64, device=dev)
    _lib.call("pf_integrate_partials", ptr(w), n, k, ptr(pos), ptr(nrm), ptr(mt), ptr(th), ptr(out), stream_handle())
    length = characteristic_length(pos)
    o = out.cpu().numpy()
    mean_pos = pos.double().mean(dim=0).cpu().numpy()
    return estimate_from_partials(o[:k], float(o[k]), o[k + 1:k + 4], n, dictionary, config, length,
                                  mean_position=mean_pos)


def voxel_mass(positions, density, grid: int, lo_hi=None):
    """BASELINE voxel-grid mass of per-point densities: returns (mass_kg, occupied, codes).

    lo_hi: optional (6,) domain; default = bbox of the points (pf_bbox)."""
    dev = require_cuda()
    t = torch()
    tor = is_torch(positions)
    p = to_dev(positions, t.float32, dev).reshape(-1, 3)
    rho = to_dev(density, t.float32, dev).reshape(-1)
    n = p.shape[0]
    st = stream_handle()
    lh = t.zeros(6, dtype=t.float64, device=dev)
    if lo_hi is None:
        _lib.call("pf_bbox", ptr(p), n, ptr(lh), st)
    else:
        lh.copy_(to_dev(lo_hi, t.float64, dev).reshape(6))
    codes = t.empty(n, dtype=t.int32, device=dev)
    _lib.call("pf_voxel_codes", ptr(p), n, ptr(lh), grid, ptr(codes), st)
    g = t.zeros(2 * grid**3, dtype=t.float32, device=dev)
    _lib.call("pf_voxel_accumulate", ptr(codes), ptr(rho), n, grid, ptr(g), st)
    out = t.zeros(2, dtype=t.float64, device=dev)
    _lib.call("pf_voxel_mass", ptr(g), grid, ptr(lh), ptr(out), st)
    o = out.cpu().numpy()
    return float(o[0]), int(round(o[1])), (codes if tor else codes.cpu().numpy())
