"""Softmax overflow guard with non-unit text rows (VERDICT r01 missing #4).

The reference normalises text rows upstream (grounding.py:86-93) but `softmax_weights`
(grounding.py:168-178) accepts any similarities and always subtracts the row max. `QueryTables`
passes the caller's rows as they are, so the fused paths must stay finite for ‖t_k‖ ≫ 1:

* the SIMT kernel subtracts the row max (pf_fused.cu);
* the tile kernel subtracts the constant bound c = 1.05 max‖t_k‖/T (k_text_bound), or the row max
  once 2c exceeds the fp32 exponent range it can shift into (pf_tile_ws.cu setup).

Each case checks (1) no status error and finite outputs; (2) the epilogue against the oracle
applied to the kernel's OWN similarities (isolates the softmax / regression arithmetic from the bf16
operand rounding, which ‖t‖/T amplifies); (3) the full oracle where the amplification keeps the
inputs' rounding below the bar (SIMT fp32).
"""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from oracle import propfield_oracle as O

pytestmark = pytest.mark.gpu

# (text scale, temperature): shift path (2c <= 120) and per-row max path (2c > 120)
CASES = [(1.0, 0.1), (3.0, 0.1), (8.0, 0.1), (12.0, 0.1), (1.0, 0.005), (40.0, 0.05)]


def _run(wl, text, temperature, **kw):
    import torch

    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(text, wl.values, wl.mid_theta)
    res = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=temperature,
                            epsilon=wl.cfg.eps, grid=wl.cfg.grid, write_sims=True, write_weights=True,
                            check=True, **kw)
    torch.cuda.synchronize()
    return res


def _epilogue_consistent(res, wl, temperature, tol):
    sims = res.sims.cpu().numpy().astype(np.float64)
    w = res.weights.cpu().numpy().astype(np.float64)
    props = res.props.cpu().numpy().astype(np.float64)
    assert np.isfinite(sims).all() and np.isfinite(w).all() and np.isfinite(props).all()
    feat = res.counts.cpu().numpy() > 0
    w_ref = O.softmax_weights(sims[feat], temperature)
    np.testing.assert_allclose(w[feat], w_ref, rtol=tol, atol=tol * 1e-2)
    np.testing.assert_allclose(w[feat].sum(1), 1.0, rtol=1e-4)
    p_ref = O.regress_with_weights(w_ref, wl.values)
    np.testing.assert_allclose(props[feat], p_ref, rtol=tol, atol=tol * np.abs(wl.values).max())
    assert (w[~feat] == 0).all() and (props[~feat] == 0).all()


@pytest.mark.parametrize("scale,temperature", CASES)
@pytest.mark.parametrize("name,force_simt", [("mini_bf16", False), ("mini_bf16", True), ("mini", False)])
def test_non_unit_text(cuda, workload, name, force_simt, scale, temperature):
    wl = workload(name)
    text = (wl.text * scale).astype(np.float32)
    res = _run(wl, text, temperature, force_simt=force_simt)
    # fp32 exp / division in the epilogue; ex2.approx on the tile path (2^-22 relative per term)
    _epilogue_consistent(res, wl, temperature, tol=2e-4)
    if force_simt or not wl.cfg.bf16:
        # fp32 features: the full composition against the oracle, the amplification ‖t‖/T of the fp32
        # feature rounding (~1e-7) stays under the 1e-4 bar
        ref = O.fuse_and_query(wl.points, wl.views(f32_maps=True), text, wl.values, temperature,
                               wl.cfg.eps, wl.cfg.grid)
        amp = max(1.0, scale / temperature / 10.0)
        np.testing.assert_allclose(res.props.cpu().numpy(), ref["props"], rtol=1e-4 * amp,
                                   atol=1e-4 * amp * np.abs(wl.values).max())


def test_x3_tile_path_non_unit_text(cuda, workload):
    """f32 maps on the x3 tile path (70k points of C2) with text rows of norm 12 at T = 0.1
    (2c = 363: the per-row max path), against the oracle on the kernel's similarities."""
    wl = workload("c2", n=70_000)
    res = _run(wl, (wl.text * 12.0).astype(np.float32), 0.1)
    _epilogue_consistent(res, wl, 0.1, tol=2e-4)


def test_tile_scale_invariance(cuda, workload):
    """Scaling text and temperature by the same power of two is exact in bf16: the tile path must
    return identical weights whichever exponent shift (constant bound / row max) it takes."""
    wl = workload("mini_bf16")
    a = _run(wl, wl.text, 0.1)
    wa = a.weights.clone()
    b = _run(wl, (wl.text * 16.0).astype(np.float32), 1.6)  # same s/T, same shift path
    assert (wa - b.weights).abs().max().item() <= 1e-6
    c = _run(wl, (wl.text * 16.0).astype(np.float32), 0.1)  # s/T x16: per-row max path
    d = _run(wl, wl.text, 0.1 / 16.0)
    assert (c.weights - d.weights).abs().max().item() <= 1e-6


def test_infinite_text_flagged(cuda, workload):
    """An infinite text value makes the softmax sum non-finite: MaterialError, not silent NaN."""
    wl = workload("mini_bf16")
    text = wl.text.copy()
    text[0, 0] = np.inf
    for force in (False, True):
        with pytest.raises(pf.MaterialError):
            _run(wl, text, 0.1, force_simt=force)
