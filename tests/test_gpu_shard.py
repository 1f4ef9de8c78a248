"""Cell-range sharding on the device kernels (csrc/pf_shard.cu + dist.cell_sharded_steps), with W
virtual ranks on one GPU driven by the in-process loopback driver (`dist.run_loopback`): every
collective is a host-side step between the ranks' kernel launches, so no kernel waits on another
rank. Checked against the single-rank fused path on the same points:

* masks, visible counts, voxel codes: exact; properties: the path's bar (tile-path results depend
  on tile membership through the bilinear-weight expansion point, so 1e-2 in bf16 mode);
* reduced partials and voxel mass: equal to the single call's to f32 atomic-order rounding;
* owners' voxel sets are disjoint, every point is computed exactly once, the load is balanced;
* the device keys / cuts agree with the numpy restatements in tests/test_dist_cells.py.
"""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
from paper_2511_03126_b200 import _lib
from paper_2511_03126_b200 import dist as pdist
from test_dist_cells import BINS, cell_axes, cuts_ref

pytestmark = pytest.mark.gpu


def _device_inputs(wl):
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
    return views, tables


def _run_sharded(wl, views, tables, world, points=None):
    import torch

    pts_all = wl.points if points is None else points
    n = pts_all.shape[0]
    gens, opss = [], []
    for r in range(world):
        lo, hi = pdist.shard_range(n, r, world)
        pts = torch.from_numpy(np.ascontiguousarray(pts_all[lo:hi])).cuda()
        ops = pdist.DeviceShardOps(views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps,
                                   grid=wl.cfg.grid)
        opss.append(ops)
        gens.append(pdist.cell_sharded_steps(pts, r, world, ops, k=tables.k, p=tables.p,
                                             nwords=(views.nviews + 31) // 32))
    res = pdist.run_loopback(gens)
    torch.cuda.synchronize()
    return res, opss


def _check(wl, views, tables, world, tol, points=None):
    import torch

    pts_all = wl.points if points is None else points
    one = pf.fuse_and_query(torch.from_numpy(np.ascontiguousarray(pts_all)).cuda(), views, tables,
                            temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid, check=True)
    res, opss = _run_sharded(wl, views, tables, world, points)
    cat = lambda f: torch.cat([f(r) for r in res])  # noqa: E731
    assert torch.equal(cat(lambda r: r.counts), one.counts)
    assert torch.equal(cat(lambda r: r.codes), one.codes)
    assert torch.equal(cat(lambda r: r.mask_bits), one.mask_bits)
    props, ref = cat(lambda r: r.props).double(), one.props.double()
    feat = one.counts > 0
    rel = ((props[:, 0] - ref[:, 0]).abs() / ref[:, 0].abs().clamp_min(1e-30))[feat]
    assert float(rel.max()) <= tol
    assert sum(r.received for r in res) == pts_all.shape[0]
    for r in res[1:]:
        assert torch.equal(r.partials, res[0].partials) and torch.equal(r.mass, res[0].mass)
    assert res[0].mass_kg() == pytest.approx(one.mass_kg(), rel=max(1e-5, tol / 10))
    assert res[0].occupied_voxels() == int(round(float(one.mass[1].item())))
    k = tables.k
    np.testing.assert_allclose(res[0].partials[:k].cpu().numpy(), one.partials[:k].cpu().numpy(),
                               rtol=max(1e-5, tol), atol=1e-6 * pts_all.shape[0])
    assert res[0].host_partials()["visible_pairs"] == int(round(float(one.partials[k + 5].item())))
    # disjoint voxel ownership: the codes of the points each rank computed
    owned = [set(ops._bufs.codes.cpu().numpy().tolist()) if ops._bufs is not None else set() for ops in opss]
    for a in range(world):
        for b in range(a + 1, world):
            assert not (owned[a] & owned[b]), "two ranks own the same voxel"
    sizes = [r.received for r in res]
    assert max(sizes) <= pts_all.shape[0] / world * 1.25 + 256, sizes


@pytest.mark.parametrize("name,world", [("mini", 2), ("mini", 3), ("mini_bf16", 2), ("mini_bf16", 4)])
def test_loopback_small(cuda, workload, name, world):
    wl = workload(name)
    views, tables = _device_inputs(wl)
    tol = 1e-2 if wl.cfg.bf16 else 1e-4
    _check(wl, views, tables, world, tol)


@pytest.mark.parametrize("name,world", [("c3", 4), ("c5", 8)])
def test_loopback_large_shapes(cuda, workload, name, world):
    """Real C3 / C5 view, map and material shapes on 200k points (tile path), 4 / 8 virtual ranks."""
    wl = workload(name, n=200_000)
    views, tables = _device_inputs(wl)
    _check(wl, views, tables, world, 1e-2)


def test_device_keys_nest_voxels_and_cuts_match(cuda, workload):
    """pf_shard_keys: points of one voxel share one key; the device histogram's cuts equal the numpy
    restatement; owners' voxel sets are disjoint."""
    import torch

    wl = workload("c2", n=100_000)
    pts = torch.from_numpy(wl.points).cuda()
    views, tables = _device_inputs(wl)
    ops = pdist.DeviceShardOps(views, tables, grid=wl.cfg.grid)
    lo_hi = ops.bbox(pts)
    keys, hist = ops.keys(pts, lo_hi)
    assert hist.numel() == BINS == int(_lib.load().pf_shard_bins())
    k = keys.cpu().numpy()[: wl.cfg.n]
    h = hist.cpu().numpy()
    assert int(h.sum()) == wl.cfg.n
    np.testing.assert_array_equal(np.bincount(k, minlength=BINS), h)
    lh = lo_hi.cpu().numpy()
    codes, _ = cell_axes(wl.points, wl.cfg.grid, lh[:3], lh[3:])
    order = np.argsort(codes, kind="stable")
    c_sorted, k_sorted = codes[order], k[order]
    same = c_sorted[1:] == c_sorted[:-1]
    assert np.array_equal(k_sorted[1:][same], k_sorted[:-1][same]), "a voxel spans two cells"
    for world in (1, 2, 3, 8, 64):
        cuts = ops.cuts(hist, world).cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(cuts, cuts_ref(h, world))
        owner = np.searchsorted(cuts[1:world], k, side="right")
        per_voxel = {}
        for c, o in zip(codes.tolist(), owner.tolist()):
            assert per_voxel.setdefault(c, o) == o
        sizes = np.bincount(owner, minlength=world)
        assert sizes.max() <= wl.cfg.n / world + h.max() + 1
    # pack: destination blocks contiguous in rank order, local indices a permutation
    cuts_t = ops.cuts(hist, 4)
    send, counts = ops.pack(pts, keys, cuts_t, 4)
    s = send.cpu().numpy()
    idx = s[:, 3].view(np.int32)
    assert np.array_equal(np.sort(idx), np.arange(wl.cfg.n))
    np.testing.assert_array_equal(s[:, :3], wl.points[idx])
    owner = np.searchsorted(cuts_t.cpu().numpy().astype(np.int64)[1:4], k[idx], side="right")
    assert np.all(np.diff(owner) >= 0)
    np.testing.assert_array_equal(np.bincount(owner, minlength=4), counts.cpu().numpy())


def test_loopback_empty_rank(cuda, workload):
    """More ranks than occupied cells' worth of points: some ranks own nothing; results still exact."""
    wl = workload("mini")
    views, tables = _device_inputs(wl)
    pts = np.ascontiguousarray(wl.points[:5])
    res, _ = _run_sharded(wl, views, tables, 8, points=pts)
    assert sum(r.received for r in res) == 5
    assert any(r.received == 0 for r in res)
    import torch

    one = pf.fuse_and_query(torch.from_numpy(pts).cuda(), views, tables, temperature=wl.cfg.temperature,
                            epsilon=wl.cfg.eps, grid=wl.cfg.grid)
    assert torch.equal(torch.cat([r.counts for r in res]), one.counts)
    assert res[0].mass_kg() == pytest.approx(one.mass_kg(), rel=1e-6)


# ---- fixed-capacity exchange (no host synchronisation) -------------------------------------------
def _padded_gens(wl, views, tables, world, capacity=None, fixed_domain=False, opss=None):
    import torch

    n = wl.points.shape[0]
    lo_hi = None
    if fixed_domain:
        p64 = wl.points.astype(np.float64)
        lo_hi = torch.from_numpy(np.concatenate([p64.min(0), p64.max(0)])).cuda()
    gens, opss = [], opss or [pdist.DeviceShardOps(views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps,
                                                   grid=wl.cfg.grid) for _ in range(world)]
    for r in range(world):
        lo, hi = pdist.shard_range(n, r, world)
        pts = torch.from_numpy(np.ascontiguousarray(wl.points[lo:hi])).cuda()
        cap = capacity or pdist.padded_capacity(hi - lo, world)
        gens.append(pdist.cell_sharded_steps_padded(pts, r, world, opss[r], k=tables.k, p=tables.p,
                                                    nwords=(views.nviews + 31) // 32, capacity=cap, lo_hi=lo_hi))
    return gens, opss


@pytest.mark.parametrize("name,world,fixed", [("mini", 2, False), ("mini_bf16", 3, True), ("c5", 8, True)])
def test_padded_exchange_loopback(cuda, workload, name, world, fixed):
    """The graph-capturable protocol on the device kernels: results equal the single call's."""
    import torch

    wl = workload(name, n=200_000) if name == "c5" else workload(name)
    views, tables = _device_inputs(wl)
    tol = 1e-2 if wl.cfg.bf16 else 1e-4
    one = pf.fuse_and_query(torch.from_numpy(wl.points).cuda(), views, tables, temperature=wl.cfg.temperature,
                            epsilon=wl.cfg.eps, grid=wl.cfg.grid, check=True)
    gens, _ = _padded_gens(wl, views, tables, world, fixed_domain=fixed)
    res = pdist.run_loopback(gens)
    torch.cuda.synchronize()
    assert not any(r.overflowed() for r in res)
    cat = lambda f: torch.cat([f(r) for r in res])  # noqa: E731
    assert torch.equal(cat(lambda r: r.counts), one.counts)
    assert torch.equal(cat(lambda r: r.codes), one.codes)
    assert torch.equal(cat(lambda r: r.mask_bits), one.mask_bits)
    feat = one.counts > 0
    props, ref = cat(lambda r: r.props).double(), one.props.double()
    rel = ((props[:, 0] - ref[:, 0]).abs() / ref[:, 0].abs().clamp_min(1e-30))[feat]
    assert float(rel.max()) <= tol
    assert res[0].mass_kg() == pytest.approx(one.mass_kg(), rel=max(1e-5, tol / 10))
    assert res[0].occupied_voxels() == int(round(float(one.mass[1].item())))


def test_padded_exchange_overflow_flagged_on_device(cuda, workload):
    import torch

    wl = workload("mini")
    views, tables = _device_inputs(wl)
    gens, _ = _padded_gens(wl, views, tables, 2, capacity=16)
    res = pdist.run_loopback(gens)
    torch.cuda.synchronize()
    assert all(r.overflowed() for r in res)


def test_padded_step_cuda_graph_capture(cuda, workload):
    """The fixed-capacity sharded step (2 loopback ranks, fixed domain) captured in one CUDA graph
    and replayed: no host synchronisation inside, same results as the eager step."""
    import torch

    wl = workload("mini_bf16")
    views, tables = _device_inputs(wl)
    gens, opss = _padded_gens(wl, views, tables, 2, fixed_domain=True)
    eager = pdist.run_loopback(gens)  # warm-up: buffers and workspaces allocated at capacity
    torch.cuda.synchronize()
    ref = [(r.counts.clone(), r.codes.clone(), r.props.clone(), r.mass.clone()) for r in eager]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        gens, _ = _padded_gens(wl, views, tables, 2, fixed_domain=True, opss=opss)
        with torch.cuda.graph(g, stream=s):
            out = pdist.run_loopback(gens)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for r, (c, k, pr, m) in zip(out, ref):
        assert torch.equal(r.counts, c) and torch.equal(r.codes, k)
        assert torch.allclose(r.props, pr, rtol=1e-6, atol=1e-5)
        assert float(r.mass[0]) == pytest.approx(float(m[0]), rel=1e-6)


def test_nan_points_are_inert_padding(cuda, workload):
    """NaN points (padding slots of the fixed-capacity exchange): no view, code -1, zero outputs,
    no effect on the mass or partials, on both the SIMT and the tensor-core paths."""
    import torch

    for name in ("mini", "mini_bf16"):
        wl = workload(name)
        views, tables = _device_inputs(wl)
        pts = wl.points
        pad = np.full((300, 3), np.nan, np.float32)
        mixed = np.concatenate([pts[:700], pad[:150], pts[700:], pad[150:]])
        p64 = pts.astype(np.float64)
        lo_hi = np.concatenate([p64.min(0), p64.max(0)])
        kw = dict(temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid, lo_hi=lo_hi, check=True)
        a = pf.fuse_and_query(torch.from_numpy(pts).cuda(), views, tables, **kw)
        ac, am, ap = a.counts.clone(), a.mass_kg(), a.partials.clone()
        b = pf.fuse_and_query(torch.from_numpy(mixed).cuda(), views, tables, **kw)
        real = ~np.isnan(mixed[:, 0])
        assert torch.equal(b.counts[torch.from_numpy(real).cuda()], ac)
        assert (b.counts[torch.from_numpy(~real).cuda()] == 0).all()
        assert (b.codes[torch.from_numpy(~real).cuda()] == -1).all()
        assert (b.props[torch.from_numpy(~real).cuda()] == 0).all()
        assert (b.mask_bits[torch.from_numpy(~real).cuda()] == 0).all()
        # the tile path's weights depend on which points share a 32-row group (the expansion centre):
        # padding rows shift the groups, so the bf16 path agrees at its bar, the SIMT path exactly
        tol = 1e-2 if wl.cfg.bf16 else 1e-5
        assert b.mass_kg() == pytest.approx(am, rel=tol)
        torch.testing.assert_close(b.partials, ap, rtol=tol, atol=1e-6)


def test_allreduce_partials_nccl_entry(cuda):
    """pf_allreduce_partials over a one-rank NCCL communicator (the C entry a C/C++ host calls with
    its own ncclComm_t): an identity sum, in place, on the stream."""
    import ctypes as C

    import torch

    from paper_2511_03126_b200.device import stream_handle

    lib = _lib.load()
    comm = C.c_void_p()
    _lib.check(lib.pf_nccl_comm_init_single(C.byref(comm)))
    try:
        grid = torch.arange(1000, dtype=torch.float32, device="cuda")
        part = torch.linspace(0, 1, 70, dtype=torch.float64, device="cuda")
        g0, p0 = grid.clone(), part.clone()
        _lib.call("pf_allreduce_partials", grid.data_ptr(), grid.numel(), part.data_ptr(), part.numel(), comm.value,
                  stream_handle())
        torch.cuda.synchronize()
        assert torch.equal(grid, g0) and torch.equal(part, p0)
        with pytest.raises(ValueError):
            _lib.call("pf_allreduce_partials", grid.data_ptr(), 10, part.data_ptr(), 1, None, stream_handle())
    finally:
        _lib.check(lib.pf_nccl_comm_destroy(comm.value))
