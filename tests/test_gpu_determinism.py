"""Race evidence for the warp-specialised kernels (compute-sanitizer is closed on
this GPU pool, see profiles/r02_checked_builds.md).

Every work item of the tile kernels is processed start to finish by one CTA with fixed roles, so
its per-point outputs must not depend on how items are spread over CTAs or on timing. A missing
barrier, a TMEM / shared-memory slot reused before it was read, or an mbarrier phase error would
show up as run-to-run or grid-size-dependent differences. These tests run the same objects with
different persistent-grid sizes (PF_WS_GRID: 148, 37, 5 CTAs, i.e. 1 to ~30 items per CTA and
different role interleavings) and require BIT-IDENTICAL masks, counts, codes, properties and
similarities; the voxel mass is a sum of fp32 atomics and is compared at 1e-6. The runs use
PF_FUSE_DETERMINISTIC (stable point sort): the default counting sort orders the points of one sort
cell differently from run to run, which moves a few points between tiles (a ~1e-6 effect).
"""

import os

import numpy as np
import pytest

import paper_2511_03126_b200 as pf

pytestmark = pytest.mark.gpu


def _run(wl, grid_ctas, **kw):
    import torch

    os.environ["PF_WS_GRID"] = str(grid_ctas)
    try:
        views = pf.ViewSet.from_views(wl.views())
        tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
        r = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=wl.cfg.temperature,
                              epsilon=wl.cfg.eps, grid=wl.cfg.grid, write_sims=True, check=True, deterministic=True,
                              **kw)
        torch.cuda.synchronize()
        return {k: getattr(r, k).cpu().numpy().copy() for k in ("counts", "codes", "mask_bits", "props", "sims")}, \
            r.mass_kg()
    finally:
        os.environ.pop("PF_WS_GRID", None)


@pytest.mark.parametrize("name,n,kw", [("mini_bf16", None, {}), ("c5", 60_000, {}), ("c3", 60_000, {}),
                                       ("c5", 30_000, {"feature_kernel": True}), ("c2", 70_000, {})])
def test_grid_size_invariance(cuda, workload, name, n, kw):
    wl = workload(name, n=n) if n else workload(name)
    base, mass = _run(wl, 148, **kw)
    for ctas in (37, 5, 148):
        out, m = _run(wl, ctas, **kw)
        for k in base:
            assert np.array_equal(out[k], base[k]), f"{name}: {k} differs with {ctas} CTAs"
        assert m == pytest.approx(mass, rel=1e-6)


def _tables(wl):
    return pf.ViewSet.from_views(wl.views()), pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)


@pytest.mark.parametrize("name,n,kw", [("c5", 60_000, {}), ("c3", 60_000, {}),
                                       ("c5", 30_000, {"feature_kernel": True}), ("c2", 70_000, {})])
def test_forked_prepare_matches_serial(cuda, workload, name, n, kw):
    """pf_fuse_query builds the G table on a forked stream (joined before the tensor-core kernel);
    the outputs must be bit-identical to the serial pf_fuse_prepare + PF_FUSE_PREPARED call."""
    import torch

    wl = workload(name, n=n)
    views, tables = _tables(wl)
    pts = torch.from_numpy(wl.points).cuda()
    common = dict(temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid, write_sims=True,
                  check=True, deterministic=True, **kw)
    forked = pf.fuse_and_query(pts, views, tables, **common)
    f = {k: getattr(forked, k).cpu().numpy().copy() for k in ("counts", "codes", "mask_bits", "props", "sims")}
    mf = forked.mass_kg()
    bufs = pf.FuseBuffers(pts.shape[0], views, tables, wl.cfg.grid, sims=True)
    pf.fuse_prepare(views, tables, bufs)
    serial = pf.fuse_and_query(pts, views, tables, buffers=bufs, prepared=True, reset=False, **common)
    for k in f:
        assert np.array_equal(getattr(serial, k).cpu().numpy(), f[k]), f"{name}: {k} differs"
    assert serial.mass_kg() == pytest.approx(mf, rel=1e-6)


def test_forked_prepare_graph_capture(cuda, workload):
    """The fork / join of the G-table stream is event based, so a captured step replays the whole
    path: the replay over fresh buffers reproduces the eager call bit for bit."""
    import torch

    wl = workload("c5", n=40_000)
    views, tables = _tables(wl)
    pts = torch.from_numpy(wl.points).cuda()
    common = dict(temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid, deterministic=True,
                  reduce=False)
    eager_bufs = pf.FuseBuffers(pts.shape[0], views, tables, wl.cfg.grid)
    eager = pf.fuse_and_query(pts, views, tables, buffers=eager_bufs, **common)
    want = {k: getattr(eager, k).cpu().numpy().copy() for k in ("counts", "codes", "mask_bits", "props")}
    bufs = pf.FuseBuffers(pts.shape[0], views, tables, wl.cfg.grid)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up on the capture stream (creates the forked stream)
        pf.fuse_and_query(pts, views, tables, buffers=bufs, **common)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    bufs.props.zero_()
    bufs.counts.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        res = pf.fuse_and_query(pts, views, tables, buffers=bufs, reset=False, **common)
    bufs.props.fill_(-1.0)
    bufs.counts.fill_(-1)
    g.replay()
    torch.cuda.synchronize()
    for k in want:
        assert np.array_equal(getattr(res, k).cpu().numpy(), want[k]), f"graph replay: {k} differs"
