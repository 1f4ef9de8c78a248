"""Point-range sharding across ranks — host logic on CPU with gloo, world_size 2.

Each rank takes its contiguous point range, agrees on the global voxel domain through
`dist.global_bbox`, computes its dense voxel partials and integrate_mass partials (here with the
CPU oracle standing in for the device kernel — same partial layout as pf_fuse_query), then
`dist.allreduce_partials` sums them. The merged mass and partials must equal the single-process
result on all points.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import propfield_oracle as O
from paper_2511_03126_b200 import dist as pdist
from paper_2511_03126_b200 import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partials(points, views, wl, lo, hi):
    """One rank's partials: dense [sum rho | count] grid (f32) + [weight totals, pm, pm*x, ...]."""
    g = wl.cfg.grid
    out = O.fuse_and_query(points, views, wl.text, wl.values, wl.cfg.temperature, wl.cfg.eps, g)
    codes, _ = O.voxel_codes(points, g, lo, hi)
    grid = np.zeros(2 * g**3, dtype=np.float32)
    np.add.at(grid, codes, out["props"][:, 0].astype(np.float32))
    np.add.at(grid, g**3 + codes, 1.0)
    w = out["weights"]
    pm = w @ wl.mid_theta
    p = points.astype(np.float64)
    part = np.concatenate([w.sum(0), [pm.sum()], (pm[:, None] * p).sum(0),
                           [(out["counts"] > 0).sum(), out["counts"].sum()]])
    return grid, part


def _mass_from_grid(grid, g, lo, hi):
    edge = float((np.asarray(hi) - np.asarray(lo)).max()) / g
    s, c = grid[: g**3].astype(np.float64), grid[g**3 :].astype(np.float64)
    occ = c > 0
    return edge**3 * float((s[occ] / c[occ]).sum()), int(occ.sum())


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.generate("mini")
        lo_i, hi_i = pdist.shard_range(wl.cfg.n, rank, world)
        pts = wl.points[lo_i:hi_i]
        lo_hi = torch.tensor(np.concatenate([pts.min(0), pts.max(0)]).astype(np.float64))
        pdist.global_bbox(lo_hi)
        lo, hi = lo_hi[:3].numpy(), lo_hi[3:].numpy()
        grid, part = _partials(pts, wl.views(f32_maps=True), wl, lo, hi)
        tg, tp = torch.from_numpy(grid), torch.from_numpy(part)
        pdist.allreduce_partials(tg, tp)
        mass, occ = _mass_from_grid(tg.numpy(), wl.cfg.grid, lo, hi)
        q.put((rank, lo_hi.numpy(), tp.numpy(), mass, occ))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_and_balance():
    for n in (0, 1, 7, 1000, 16_000_000):
        for w in (1, 2, 3, 8):
            rs = [pdist.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pdist.shard_range(10, 2, 2)


def test_two_rank_partials_match_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # every rank agrees on the domain and the reduced partials
    assert np.array_equal(res[0][1], res[1][1])
    np.testing.assert_array_equal(res[0][2], res[1][2])
    # ... and they equal the single-process oracle on all points
    wl = workloads.generate("mini")
    lo, hi = O.voxel_domain(wl.points)
    np.testing.assert_array_equal(res[0][1], np.concatenate([lo, hi]))
    grid, part = _partials(wl.points, wl.views(f32_maps=True), wl, lo, hi)
    np.testing.assert_allclose(res[0][2], part, rtol=1e-12)
    mass, occ = _mass_from_grid(grid, wl.cfg.grid, lo, hi)
    assert res[0][4] == occ
    assert res[0][3] == pytest.approx(mass, rel=1e-6)
    ref = O.fuse_and_query(wl.points, wl.views(f32_maps=True), wl.text, wl.values,
                           wl.cfg.temperature, wl.cfg.eps, wl.cfg.grid)
    assert res[0][3] == pytest.approx(ref["mass"], rel=1e-5)
