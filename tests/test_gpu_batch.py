"""Batched objects (BASELINE config 4; batch.fuse_batch): each object's packed outputs equal a
separate fuse_and_query call on it (same kernels: masks / counts / codes / properties exact, mass to
f32 atomic-order rounding), and against the CPU oracle at the fp32 bar."""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from oracle import propfield_oracle as O
from paper_2511_03126_b200 import workloads

pytestmark = pytest.mark.gpu


def _objects(name, seeds, n=None):
    wls = [workloads.generate(name, seed=s, n=n) for s in seeds]
    views = [pf.ViewSet.from_views(w.views()) for w in wls]
    tables = [pf.QueryTables.build(w.text, w.values, w.mid_theta) for w in wls]
    return wls, views, tables


@pytest.mark.parametrize("name,seeds,n,streams", [("mini", [0, 1, 2], None, 2), ("c4", [10, 11, 12, 13], 20_000, 3),
                                                  ("mini_bf16", [3, 4], None, 1)])
def test_batch_equals_single_calls(cuda, name, seeds, n, streams):
    import torch

    wls, views, tables = _objects(name, seeds, n)
    pts = [torch.from_numpy(w.points).cuda() for w in wls]
    res, ws = pf.fuse_batch(pts, views, tables, temperature=wls[0].cfg.temperature, epsilon=wls[0].cfg.eps,
                            grid=wls[0].cfg.grid, streams=streams)
    torch.cuda.synchronize()
    for i, w in enumerate(wls):
        one = pf.fuse_and_query(pts[i], views[i], tables[i], temperature=w.cfg.temperature, epsilon=w.cfg.eps,
                                grid=w.cfg.grid)
        a, b = res.offsets[i], res.offsets[i + 1]
        assert torch.equal(res.counts[a:b], one.counts)
        assert torch.equal(res.codes[a:b], one.codes)
        assert torch.equal(res.mask_bits[a:b], one.mask_bits)
        tol = 1e-2 if w.cfg.bf16 else 1e-5
        torch.testing.assert_close(res.props[a:b], one.props, rtol=tol, atol=tol)
        assert float(res.mass[i, 0]) == pytest.approx(one.mass_kg(), rel=1e-5)
        assert float(res.mass[i, 1]) == float(one.mass[1])
        if name == "mini":  # and the oracle at the fp32 bar
            ref = O.fuse_and_query(w.points, w.views(f32_maps=True), w.text, w.values, w.cfg.temperature,
                                   w.cfg.eps, w.cfg.grid)
            np.testing.assert_array_equal(res.counts[a:b].cpu().numpy(), ref["counts"])
            np.testing.assert_allclose(res.props[a:b].cpu().numpy(), ref["props"], rtol=1e-4, atol=1e-6)
            assert float(res.mass[i, 0]) == pytest.approx(ref["mass"], rel=1e-4)
    # the workspace is reusable for a second batch of the same shapes
    res2, ws2 = pf.fuse_batch(pts, views, tables, temperature=wls[0].cfg.temperature, epsilon=wls[0].cfg.eps,
                              grid=wls[0].cfg.grid, streams=streams, workspace=ws)
    torch.cuda.synchronize()
    assert ws2 is ws
    assert torch.equal(res2.counts, res.counts)
    torch.testing.assert_close(res2.mass, res.mass, rtol=1e-5, atol=0)


def test_batch_mixed_sizes_and_views(cuda):
    """Objects of different sizes and view counts in one batch (narrower mask rows are widened)."""
    import torch

    a = workloads.generate("mini", seed=5, n=700)
    b = workloads.generate("mini_fib40", seed=6)
    wa, wb = (pf.ViewSet.from_views(w.views()) for w in (a, b))
    # same D / K / P for the packed outputs: rebuild b's tables with a's K rows at b's D
    rng = np.random.default_rng(0)
    tb_text = rng.standard_normal((a.text.shape[0], b.cfg.d)).astype(np.float32)
    tb_text /= np.linalg.norm(tb_text, axis=1, keepdims=True)
    ta = pf.QueryTables.build(a.text, a.values, a.mid_theta)
    tb = pf.QueryTables.build(tb_text, a.values, a.mid_theta)
    pts = [torch.from_numpy(a.points).cuda(), torch.from_numpy(b.points).cuda()]
    res, _ = pf.fuse_batch(pts, [wa, wb], [ta, tb], grid=16, streams=2)
    torch.cuda.synchronize()
    for i, (p, v, t) in enumerate(zip(pts, (wa, wb), (ta, tb))):
        one = pf.fuse_and_query(p, v, t, grid=16)
        lo, hi = res.offsets[i], res.offsets[i + 1]
        assert torch.equal(res.counts[lo:hi], one.counts)
        w = one.mask_bits.shape[1]
        assert torch.equal(res.mask_bits[lo:hi, :w], one.mask_bits)
        assert float(res.mass[i, 0]) == pytest.approx(one.mass_kg(), rel=1e-5)
