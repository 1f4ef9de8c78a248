"""Cell-range sharding (SURVEY §8e alternative; csrc/pf_shard.cu) — the rank-local protocol
`dist.cell_sharded_steps` driven by real gloo collectives on CPU (world_size 2 and 3) and by the
in-process loopback driver.

The rank-local steps run through `CpuShardOps` below: numpy restatements of the pf_shard_* kernels
(cell keys derived from the voxel code, balanced cuts of the global histogram, owner grouping) and
the CPU oracle for the fused pass — same data layouts as DeviceShardOps. What is checked here is
the protocol: every point reaches exactly one owner, owners' voxel sets are disjoint, the reduced
partials and voxel mass equal the single-process oracle, and every rank gets its own points'
results back in its caller order. tests/test_gpu_shard.py runs the same protocol on the device
kernels and checks `cuts_ref` / the keys against them.
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

CELL_BITS = 6
BINS = 1 << (3 * CELL_BITS)


def cuts_ref(hist: np.ndarray, world: int) -> np.ndarray:
    """pf_shard_cuts: cut_r = first bin c with exclusive prefix(c) >= ceil(r * total / world)."""
    prefix = np.concatenate([[0], np.cumsum(hist.astype(np.int64))])
    total = int(prefix[-1])
    cuts = np.empty(world + 1, dtype=np.int64)
    cuts[0], cuts[world] = 0, BINS
    for r in range(1, world):
        target = (total * r + world - 1) // world
        cuts[r] = np.searchsorted(prefix, target, side="left")
    return cuts


def cell_axes(points, grid, lo, hi):
    codes, _ = O.voxel_codes(points, grid, lo, hi)
    cx, cy, cz = codes // (grid * grid), (codes // grid) % grid, codes % grid
    return codes, [c * (1 << CELL_BITS) // grid for c in (cx, cy, cz)]


def morton_key(cells):
    """Any spatial key works for the protocol (the device uses a Hilbert key): Morton here."""
    key = np.zeros_like(cells[0])
    for b in range(CELL_BITS):
        for a in range(3):
            key |= ((cells[a] >> b) & 1) << (3 * b + (2 - a))
    return key


class CpuShardOps:
    """numpy / oracle restatement of DeviceShardOps for the CPU protocol tests."""

    def __init__(self, wl):
        self.wl = wl
        self.views = wl.views(f32_maps=True)
        self.grid = wl.cfg.grid

    def bbox(self, points):
        p = points.numpy().astype(np.float64)
        if p.shape[0] == 0:
            return torch.tensor([np.inf] * 3 + [-np.inf] * 3, dtype=torch.float64)
        return torch.from_numpy(np.concatenate([p.min(0), p.max(0)]))

    def keys(self, points, lo_hi):
        lh = lo_hi.numpy()
        _, cells = cell_axes(points.numpy(), self.grid, lh[:3], lh[3:])
        key = morton_key(cells)
        hist = np.bincount(key, minlength=BINS).astype(np.int32)
        return torch.from_numpy(key.astype(np.int32)), torch.from_numpy(hist)

    def cuts(self, hist, world):
        return torch.from_numpy(cuts_ref(hist.numpy(), world).astype(np.int32))

    def pack(self, points, keys, cuts, world):
        owner = np.searchsorted(cuts.numpy()[1:world], keys.numpy(), side="right")
        order = np.argsort(owner, kind="stable")
        p = points.numpy()
        send = np.empty((p.shape[0], 4), dtype=np.float32)
        send[:, :3] = p[order]
        send[:, 3] = order.astype(np.int32).view(np.float32)
        counts = np.bincount(owner, minlength=world).astype(np.int64)
        return torch.from_numpy(send), torch.from_numpy(counts)

    def fuse(self, recv, lo_hi):
        wl, g = self.wl, self.grid
        pts = recv.numpy()[:, :3].copy()
        lh = lo_hi.numpy()
        out = O.fuse_and_query(pts, self.views, wl.text, wl.values, wl.cfg.temperature, wl.cfg.eps, g)
        codes, edge = O.voxel_codes(pts, g, lh[:3], lh[3:])
        s = np.zeros(g**3)
        c = np.zeros(g**3)
        np.add.at(s, codes, out["props"][:, 0])
        np.add.at(c, codes, 1.0)
        occ = c > 0
        w = out["weights"]
        pm = w @ wl.mid_theta
        part = np.concatenate([w.sum(0), [pm.sum()], (pm[:, None] * pts.astype(np.float64)).sum(0),
                               [(out["counts"] > 0).sum(), out["counts"].sum()]])
        nv = len(self.views)
        nwords = (nv + 31) // 32
        bits = np.zeros((pts.shape[0], nwords), dtype=np.int64)
        for v in range(nv):
            bits[:, v // 32] |= out["visibility"][:, v].astype(np.int64) << (v % 32)
        return {"props": out["props"].astype(np.float32), "counts": out["counts"].astype(np.int32),
                "codes": codes.astype(np.int32), "mask": (bits & 0xFFFFFFFF).astype(np.uint32).view(np.int32),
                "partials": torch.from_numpy(part),
                "mass": torch.tensor([edge**3 * float((s[occ] / c[occ]).sum()), float(occ.sum())],
                                     dtype=torch.float64),
                "voxels": np.unique(codes)}

    def pack_results(self, res):
        rows = np.concatenate([res["props"].view(np.int32), res["counts"][:, None], res["codes"][:, None],
                               res["mask"]], axis=1)
        self.last_voxels = res["voxels"]
        return torch.from_numpy(np.ascontiguousarray(rows))

    def unpack_results(self, rows, sent, n, p, nwords):
        r = rows.numpy()
        idx = sent.numpy()[:, 3].view(np.int32)
        out = {"props": np.zeros((n, p), np.float32), "counts": np.zeros(n, np.int32),
               "codes": np.zeros(n, np.int32), "mask_bits": np.zeros((n, nwords), np.int32)}
        out["props"][idx] = r[:, :p].view(np.float32)
        out["counts"][idx] = r[:, p]
        out["codes"][idx] = r[:, p + 1]
        out["mask_bits"][idx] = r[:, p + 2 :]
        return {k: torch.from_numpy(v) for k, v in out.items()}


class CpuPaddedOps(CpuShardOps):
    """numpy restatement of the fixed-capacity exchange (pf_shard_pack_padded / unpad /
    unpack_results_padded): blocks of capacity + 1 rows, row 0 = {count, flags} bits, NaN padding."""

    def pack_padded(self, points, keys, cuts, world, capacity):
        owner = np.searchsorted(cuts.numpy()[1:world], keys.numpy(), side="right")
        p = points.numpy()
        send = np.full((world, capacity + 1, 4), np.nan, dtype=np.float32)
        send[:, :, 3] = np.array(-1, np.int32).view(np.float32)
        flags = 0
        for o in range(world):
            idx = np.nonzero(owner == o)[0]
            if idx.size > capacity:
                flags, idx = 1, idx[:capacity]
            send[o, 1 : 1 + idx.size, :3] = p[idx]
            send[o, 1 : 1 + idx.size, 3] = idx.astype(np.int32).view(np.float32)
            send[o, 0, :] = 0.0
            send[o, 0, 0] = np.array(idx.size, np.int32).view(np.float32)
        for o in range(world):
            send[o, 0, 1] = np.array(flags, np.int32).view(np.float32)
        return torch.from_numpy(send), torch.tensor([flags], dtype=torch.int32)

    def unpad(self, recv, world, capacity):
        return recv[:, 1:, :3].reshape(world * capacity, 3).contiguous()

    def fuse_points(self, xyz, lo_hi):
        x = xyz.numpy()
        real = ~np.isnan(x[:, 0])
        d = super().fuse(torch.from_numpy(np.concatenate([x[real], np.zeros((int(real.sum()), 1), np.float32)], 1)),
                         lo_hi)
        m = x.shape[0]
        out = {"props": np.zeros((m, d["props"].shape[1]), np.float32), "counts": np.zeros(m, np.int32),
               "codes": np.full(m, -1, np.int32), "mask": np.zeros((m, d["mask"].shape[1]), np.int32)}
        for key in out:
            out[key][real] = d[key]
        out.update(partials=d["partials"], mass=d["mass"], voxels=d["voxels"])
        self.real_slots = int(real.sum())
        return _Res(out)

    def pack_results(self, res):
        return CpuShardOps.pack_results(self, res.d)

    def unpack_results_padded(self, rows, sent, n, p, nwords, world, capacity):
        r = rows.numpy().reshape(world, capacity, -1)
        s = sent.numpy()
        out = {"props": np.zeros((n, p), np.float32), "counts": np.zeros(n, np.int32),
               "codes": np.full(n, -1, np.int32), "mask_bits": np.zeros((n, nwords), np.int32)}
        for o in range(world):
            cnt = int(s[o, 0, 0:1].view(np.int32)[0])
            idx = s[o, 1 : 1 + cnt, 3].view(np.int32)
            out["props"][idx] = r[o, :cnt, :p].view(np.float32)
            out["counts"][idx] = r[o, :cnt, p]
            out["codes"][idx] = r[o, :cnt, p + 1]
            out["mask_bits"][idx] = r[o, :cnt, p + 2 :]
        return {k: torch.from_numpy(v) for k, v in out.items()}


class _Res:
    """Adapter: CpuShardOps.fuse returns a dict; the protocol reads .partials / .mass."""

    def __init__(self, d):
        self.__dict__.update(d)
        self.d = d


class _Ops(CpuShardOps):
    def fuse(self, recv, lo_hi):
        return _Res(super().fuse(recv, lo_hi))

    def pack_results(self, res):
        return super().pack_results(res.d)


def _steps(wl, rank, world):
    lo, hi = pdist.shard_range(wl.cfg.n, rank, world)
    pts = torch.from_numpy(np.ascontiguousarray(wl.points[lo:hi]))
    ops = _Ops(wl)
    gen = pdist.cell_sharded_steps(pts, rank, world, ops, k=wl.text.shape[0], p=wl.values.shape[1],
                                   nwords=(wl.cfg.nviews + 31) // 32)
    return gen, ops


def _steps_padded(wl, rank, world, capacity, fixed_domain):
    lo, hi = pdist.shard_range(wl.cfg.n, rank, world)
    pts = torch.from_numpy(np.ascontiguousarray(wl.points[lo:hi]))
    ops = CpuPaddedOps(wl)
    p64 = wl.points.astype(np.float64)
    lo_hi = torch.from_numpy(np.concatenate([p64.min(0), p64.max(0)])) if fixed_domain else None
    gen = pdist.cell_sharded_steps_padded(pts, rank, world, ops, k=wl.text.shape[0], p=wl.values.shape[1],
                                          nwords=(wl.cfg.nviews + 31) // 32, capacity=capacity, lo_hi=lo_hi)
    return gen, ops


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.generate("mini")
        gen, ops = _steps(wl, rank, world)
        res = pdist.run_dist(gen)
        q.put((rank, res.props.numpy(), res.counts.numpy(), res.codes.numpy(), res.mask_bits.numpy(),
               res.partials.numpy(), res.mass.numpy(), res.received, ops.last_voxels))
    finally:
        dist.destroy_process_group()


def _worker_padded(rank, world, port, q, capacity, fixed_domain):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.generate("mini")
        gen, ops = _steps_padded(wl, rank, world, capacity, fixed_domain)
        res = pdist.run_dist(gen)
        q.put((rank, res.props.numpy(), res.counts.numpy(), res.codes.numpy(), res.mask_bits.numpy(),
               res.partials.numpy(), res.mass.numpy(), ops.real_slots, ops.last_voxels, res.overflowed()))
    finally:
        dist.destroy_process_group()


def _single(wl):
    ref = O.fuse_and_query(wl.points, wl.views(f32_maps=True), wl.text, wl.values, wl.cfg.temperature,
                           wl.cfg.eps, wl.cfg.grid)
    return ref


def _check(wl, per_rank, world):
    ref = _single(wl)
    n = wl.cfg.n
    props = np.concatenate([r[1] for r in per_rank])
    counts = np.concatenate([r[2] for r in per_rank])
    codes = np.concatenate([r[3] for r in per_rank])
    assert props.shape[0] == n
    np.testing.assert_array_equal(counts, ref["counts"])
    np.testing.assert_array_equal(codes, ref["codes"])
    np.testing.assert_allclose(props, ref["props"], rtol=1e-6, atol=1e-4)
    vis = ref["visibility"]
    for v in range(wl.cfg.nviews):
        bit = (np.concatenate([r[4] for r in per_rank])[:, v // 32].astype(np.int64) >> (v % 32)) & 1
        np.testing.assert_array_equal(bit.astype(bool), vis[:, v])
    # every point computed exactly once, owners' voxel sets disjoint
    assert sum(r[7] for r in per_rank) == n
    vox = [set(r[8].tolist()) for r in per_rank]
    for a in range(world):
        for b in range(a + 1, world):
            assert not (vox[a] & vox[b]), "two ranks own the same voxel"
    # all ranks agree on the reduced partials and mass, which equal the single-process values
    for r in per_rank[1:]:
        np.testing.assert_array_equal(r[5], per_rank[0][5])
        np.testing.assert_array_equal(r[6], per_rank[0][6])
    assert per_rank[0][6][0] == pytest.approx(ref["mass"], rel=1e-9)
    assert int(per_rank[0][6][1]) == len(np.unique(ref["codes"]))
    k = wl.text.shape[0]
    np.testing.assert_allclose(per_rank[0][5][:k], ref["weights"].sum(0), rtol=1e-9, atol=1e-12)
    # balance: each rank computed about N / W points (cells are small at this size)
    sizes = [r[7] for r in per_rank]
    assert max(sizes) <= n / world * 1.5 + 64


@pytest.mark.parametrize("world", [2, 3])
def test_cell_sharded_gloo_matches_single_process(world):
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
    _check(workloads.generate("mini"), res, world)


@pytest.mark.parametrize("world", [1, 4])
def test_cell_sharded_loopback_matches_single_process(world):
    wl = workloads.generate("mini")
    steps = [_steps(wl, r, world) for r in range(world)]
    results = pdist.run_loopback([g for g, _ in steps])
    per_rank = [(r, x.props.numpy(), x.counts.numpy(), x.codes.numpy(), x.mask_bits.numpy(), x.partials.numpy(),
                 x.mass.numpy(), x.received, ops.last_voxels) for r, (x, (_, ops)) in enumerate(zip(results, steps))]
    _check(wl, per_rank, world)


def test_cuts_balanced_and_edge_cases():
    rng = np.random.default_rng(0)
    hist = np.zeros(BINS, np.int64)
    idx = rng.integers(0, BINS, 50_000)
    np.add.at(hist, idx, 1)
    for world in (1, 2, 7, 8, 64):
        c = cuts_ref(hist, world)
        assert c[0] == 0 and c[-1] == BINS and np.all(np.diff(c) >= 0)
        prefix = np.concatenate([[0], np.cumsum(hist)])
        sizes = prefix[c[1:]] - prefix[c[:-1]]
        assert sizes.sum() == hist.sum()
        assert sizes.max() - hist.sum() / world <= hist.max() + 1
    empty = cuts_ref(np.zeros(BINS, np.int64), 4)
    assert empty[0] == 0 and empty[-1] == BINS
    one = np.zeros(BINS, np.int64)
    one[77] = 5
    c = cuts_ref(one, 4)  # all points in one cell: exactly one rank owns it
    prefix = np.concatenate([[0], np.cumsum(one)])
    assert sorted((prefix[c[1:]] - prefix[c[:-1]]).tolist()) == [0, 0, 0, 5]


def _spawn(target, world, extra=()):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q, *extra)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    return res


@pytest.mark.parametrize("world,fixed", [(2, False), (3, True)])
def test_padded_exchange_gloo_matches_single_process(world, fixed):
    """Fixed-capacity exchange (no host synchronisation, counts in-band, NaN padding slots), with the
    union-of-bboxes or a fixed voxel domain: identical results to the single-process oracle."""
    wl = workloads.generate("mini")
    cap = pdist.padded_capacity(wl.cfg.n // world, world)
    res = _spawn(_worker_padded, world, (cap, fixed))
    assert not any(r[9] for r in res)
    _check(wl, [r[:9] for r in res], world)


def test_padded_exchange_overflow_is_flagged():
    """A capacity below one owner's share: every rank sees the overflow flag (reduced in-band)."""
    wl = workloads.generate("mini")
    world = 2
    steps = [_steps_padded(wl, r, world, 16, False) for r in range(world)]
    results = pdist.run_loopback([g for g, _ in steps])
    assert all(r.overflowed() for r in results)


@pytest.mark.parametrize("world", [1, 4])
def test_padded_exchange_loopback_matches_single_process(world):
    wl = workloads.generate("mini")
    cap = pdist.padded_capacity(wl.cfg.n // world, world)
    steps = [_steps_padded(wl, r, world, cap, True) for r in range(world)]
    results = pdist.run_loopback([g for g, _ in steps])
    per_rank = [(r, x.props.numpy(), x.counts.numpy(), x.codes.numpy(), x.mask_bits.numpy(), x.partials.numpy(),
                 x.mass.numpy(), ops.real_slots, ops.last_voxels) for r, (x, (_, ops)) in enumerate(zip(results, steps))]
    assert not any(x.overflowed() for x in results)
    _check(wl, per_rank, world)
