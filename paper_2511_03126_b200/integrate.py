"""Mass integration on the GPU: the reference's integrate_mass (integrate.py:98-167) and the
BASELINE voxel-grid mass.

The data-parallel part of integrate_mass — weight_totals_k = sum_i w_ik, the point masses
pm_i = w_i . (mid * theta) and their position moments — runs on the device (inside the fused kernel
on the fused path, or from a probability matrix here). What remains is O(K) host arithmetic in the
reference's order (integrate.py:128-155). The characteristic length L (integrate.py:72-95, a k=8
nearest-neighbour area estimate) is SURVEY §8f "next" work; until the device kNN lands it is an
input (`length=`) or computed by the caller.
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
