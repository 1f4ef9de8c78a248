"""Point-range sharding across the GPUs of one box, torch.distributed plumbing.

* Each rank owns the contiguous point range `shard_range(n, rank, world)`; views, text and the
  material table are replicated (built per GPU).
* The voxel domain must be identical on every rank: `global_bbox` all-reduces the 6-float local
  bboxes (MIN over [lo, -hi]) — one tiny collective.
* After each rank's fused pass, `allreduce_partials` sums the dense voxel grid and the
  integrate_mass partials; then any rank finalises the mass.
The same code runs on NCCL (GPU) and gloo (CPU tests); no data-path collective exists besides
these reductions.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple:
    """[r*N/W, (r+1)*N/W) — contiguous, balanced to within one point, covering [0, N)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return (n * rank) // world, (n * (rank + 1)) // world


def global_bbox(lo_hi, group=None):
    """In place: lo_hi (6,) f64 tensor [lo(3), hi(3)] -> union over ranks."""
    import torch.distributed as dist

    lo_hi[3:].neg_()
    dist.all_reduce(lo_hi, op=dist.ReduceOp.MIN, group=group)
    lo_hi[3:].neg_()
    return lo_hi


def allreduce_partials(grid_partials, partials, group=None):
    """Sum the dense voxel grid (f32 [sum | count]) and the f64 integrate partials over ranks.

    Two buffers of different dtypes -> two all-reduce calls, issued back to back on the same
    stream (the f64 one is K+6 numbers)."""
    import torch.distributed as dist

    dist.all_reduce(grid_partials, group=group)
    dist.all_reduce(partials, group=group)


# ==============================================================================================
# Cell-range sharding ("shard by voxel-code ranges after a pre-sort")
#
# Point-range sharding above needs the dense voxel all-reduce (2 G^3 floats: 1.07 GB at 512^3),
# which at 8 GPUs costs more than the fused pass itself. `cell_sharded_steps` instead routes every
# point to the rank that owns its voxel (csrc/pf_shard.cu explains the ownership rule), so voxel
# partials are rank-local and the only reductions are a 1 MB histogram and K + 8 doubles. The
# exchange is two all-to-alls over NVLink (points out, per-point results back), ~40 B per point.
#
# The rank-local algorithm is a generator that YIELDS its collectives; a driver executes them:
#   run_dist(gen, group)   torch.distributed (NCCL on GPUs, gloo in the CPU tests)
#   run_loopback(gens)     W virtual ranks in one process, collectives done as device copies
#                          (the single-GPU parity tests of the multi-rank data path; the ranks'
#                          kernels never wait on each other: every collective is a host-side step)
# Collective requests:
#   ("allreduce", tensor, "sum" | "min")            in place
#   ("alltoall", recv (W,), send (W,))              one element per peer
#   ("alltoallv", recv, send, recv_splits, send_splits)   rows along dim 0
# ==============================================================================================


class DeviceShardOps:
    """The rank-local steps on the GPU (C ABI: pf_bbox, pf_shard_*, pf_fuse_query)."""

    def __init__(self, views, tables, *, temperature=0.1, epsilon=0.01, grid=64):
        self.views, self.tables = views, tables
        self.temperature, self.epsilon, self.grid = float(temperature), float(epsilon), int(grid)
        self._bufs = None

    @staticmethod
    def _st():
        from .device import stream_handle

        return stream_handle()

    def bbox(self, points):
        from . import _lib
        from .device import torch

        t = torch()
        lo_hi = t.empty(6, dtype=t.float64, device=points.device)
        if points.shape[0] == 0:  # identity of the MIN reduction over [lo, -hi]
            lo_hi.copy_(t.tensor([float("inf")] * 3 + [float("-inf")] * 3, dtype=t.float64))
        else:
            _lib.call("pf_bbox", points.data_ptr(), points.shape[0], lo_hi.data_ptr(), self._st())
        return lo_hi

    def keys(self, points, lo_hi):
        from . import _lib
        from .device import torch

        t = torch()
        n = points.shape[0]
        keys = t.empty(max(1, n), dtype=t.int32, device=points.device)
        hist = t.zeros(int(_lib.load().pf_shard_bins()), dtype=t.int32, device=points.device)
        _lib.call("pf_shard_keys", points.data_ptr(), n, lo_hi.data_ptr(), self.grid, keys.data_ptr(),
                  hist.data_ptr(), self._st())
        return keys, hist

    def cuts(self, hist, world):
        from . import _lib
        from .device import torch

        t = torch()
        cuts = t.empty(world + 1, dtype=t.int32, device=hist.device)
        _lib.call("pf_shard_cuts", hist.data_ptr(), world, cuts.data_ptr(), self._st())
        return cuts

    def pack(self, points, keys, cuts, world):
        from . import _lib
        from .device import torch

        t = torch()
        n = points.shape[0]
        counts = t.empty(world, dtype=t.int32, device=points.device)
        cursor = t.empty(world, dtype=t.int32, device=points.device)
        send = t.empty((max(1, n), 4), dtype=t.float32, device=points.device)
        _lib.call("pf_shard_pack", points.data_ptr(), n, keys.data_ptr(), cuts.data_ptr(), world,
                  counts.data_ptr(), cursor.data_ptr(), send.data_ptr(), self._st())
        return send[:n], counts.to(t.int64)

    def fuse(self, recv, lo_hi):
        """The fused path on the received points; voxel mass over this rank's (owned) voxels."""
        from . import _lib
        from .device import torch
        from .fused import FuseBuffers, fuse_and_query

        t = torch()
        n = recv.shape[0]
        xyz = t.empty((n, 3), dtype=t.float32, device=recv.device)
        _lib.call("pf_shard_xyz", recv.data_ptr(), n, xyz.data_ptr(), self._st())
        if self._bufs is None or self._bufs.capacity < n:  # capacity: a new point count reuses them
            cap = n if self._bufs is None else max(n, int(self._bufs.capacity * 1.25))
            self._bufs = FuseBuffers(max(cap, 1), self.views, self.tables, self.grid, device=recv.device)
        res = fuse_and_query(xyz, self.views, self.tables, temperature=self.temperature, epsilon=self.epsilon,
                             grid=self.grid, lo_hi=lo_hi, buffers=self._bufs, reduce=True)
        return res

    def pack_results(self, res):
        from . import _lib
        from .device import torch

        t = torch()
        props = res.props
        n, p, nwords = props.shape[0], props.shape[1], res.mask_bits.shape[1]
        rows = t.empty((n, p + 2 + nwords), dtype=t.int32, device=props.device)
        _lib.call("pf_shard_pack_results", n, p, nwords, props.data_ptr(), res.counts.data_ptr(),
                  res.codes.data_ptr(), res.mask_bits.data_ptr(), rows.data_ptr(), self._st())
        return rows

    # ---- fixed-capacity exchange (no host synchronisation) ----------------------------------------
    def pack_padded(self, points, keys, cuts, world, capacity):
        """(world, capacity + 1, 4) f32 blocks: row 0 = {count, flags} bits, then the owner's points,
        NaN padding (pf_shard_pack_padded)."""
        from . import _lib
        from .device import torch

        t = torch()
        n = points.shape[0]
        send = t.empty((world, capacity + 1, 4), dtype=t.float32, device=points.device)
        cursor = t.empty(world, dtype=t.int32, device=points.device)
        flags = t.empty(1, dtype=t.int32, device=points.device)
        _lib.call("pf_shard_pack_padded", points.data_ptr(), n, keys.data_ptr(), cuts.data_ptr(), world, capacity,
                  cursor.data_ptr(), send.data_ptr(), flags.data_ptr(), self._st())
        return send, flags

    def unpad(self, recv, world, capacity):
        from . import _lib
        from .device import torch

        t = torch()
        xyz = t.empty((world * capacity, 3), dtype=t.float32, device=recv.device)
        _lib.call("pf_shard_unpad", recv.data_ptr(), world, capacity, xyz.data_ptr(), self._st())
        return xyz

    def fuse_points(self, xyz, lo_hi):
        """The fused path on (m, 3) points (NaN rows: padding slots)."""
        from .fused import FuseBuffers, fuse_and_query

        n = xyz.shape[0]
        if self._bufs is None or self._bufs.capacity < n:
            self._bufs = FuseBuffers(max(n, 1), self.views, self.tables, self.grid, device=xyz.device)
        return fuse_and_query(xyz, self.views, self.tables, temperature=self.temperature, epsilon=self.epsilon,
                              grid=self.grid, lo_hi=lo_hi, buffers=self._bufs, reduce=True)

    def unpack_results_padded(self, rows, sent, n, p, nwords, world, capacity):
        from . import _lib
        from .device import torch

        t = torch()
        dev = rows.device
        out = {"props": t.zeros((n, p), dtype=t.float32, device=dev), "counts": t.zeros(n, dtype=t.int32, device=dev),
               "codes": t.full((n,), -1, dtype=t.int32, device=dev),
               "mask_bits": t.zeros((n, nwords), dtype=t.int32, device=dev)}
        _lib.call("pf_shard_unpack_results_padded", world, capacity, p, nwords, rows.data_ptr(), sent.data_ptr(),
                  out["props"].data_ptr(), out["counts"].data_ptr(), out["codes"].data_ptr(),
                  out["mask_bits"].data_ptr(), self._st())
        return out

    def unpack_results(self, rows, sent, n, p, nwords):
        from . import _lib
        from .device import torch

        t = torch()
        dev = rows.device
        out = {"props": t.empty((n, p), dtype=t.float32, device=dev), "counts": t.empty(n, dtype=t.int32, device=dev),
               "codes": t.empty(n, dtype=t.int32, device=dev),
               "mask_bits": t.empty((n, nwords), dtype=t.int32, device=dev)}
        _lib.call("pf_shard_unpack_results", n, p, nwords, rows.data_ptr(), sent.data_ptr(),
                  out["props"].data_ptr(), out["counts"].data_ptr(), out["codes"].data_ptr(),
                  out["mask_bits"].data_ptr(), self._st())
        return out


class ShardedResult:
    """Outputs of one cell-sharded pass on one rank: this rank's input points in caller order, the
    global (all-reduced) partials and voxel mass."""

    def __init__(self, out, partials, mass, lo_hi, k, received, overflow=None):
        self.props, self.counts, self.codes, self.mask_bits = (out["props"], out["counts"], out["codes"],
                                                               out["mask_bits"])
        self.partials, self.mass, self.lo_hi, self.k = partials, mass, lo_hi, k
        self.received = received  # points this rank computed (owned cells); a device count when padded
        self._overflow = overflow  # padded exchange: device scalar, > 0 if any rank dropped points

    def overflowed(self) -> bool:
        """Fixed-capacity exchange only: did some owner get more points than the capacity from some
        rank (results then incomplete: re-run with a larger capacity)? Reads one device value."""
        return bool(self._overflow is not None and float(self._overflow.item()) > 0.0)

    def mass_kg(self) -> float:
        return float(self.mass[0].item())

    def occupied_voxels(self) -> int:
        return int(round(float(self.mass[1].item())))

    def host_partials(self) -> dict:
        p = self.partials.cpu().numpy()
        k = self.k
        return {"weight_totals": p[:k], "pm_sum": p[k], "pm_pos": p[k + 1 : k + 4],
                "featured": int(round(p[k + 4])), "visible_pairs": int(round(p[k + 5]))}


def cell_sharded_steps(points, rank: int, world: int, ops, *, k: int, p: int, nwords: int):
    """Generator: the rank-local protocol of csrc/pf_shard.cu; yields collective requests and
    returns a ShardedResult. `points` (n, 3) f32 are this rank's input points (any subset; the
    caller's order is kept for the outputs)."""
    import torch as t

    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    n = int(points.shape[0])
    # 1. shared voxel domain
    lo_hi = ops.bbox(points)
    lo_hi[3:].neg_()
    yield ("allreduce", lo_hi, "min")
    lo_hi[3:].neg_()
    # 2. cell keys + global histogram -> identical cuts on every rank
    keys, hist = ops.keys(points, lo_hi)
    yield ("allreduce", hist, "sum")
    cuts = ops.cuts(hist, world)
    # 3. points to their owners
    send, counts = ops.pack(points, keys, cuts, world)
    recv_counts = t.empty_like(counts)
    yield ("alltoall", recv_counts, counts)
    send_splits = [int(x) for x in counts.tolist()]
    recv_splits = [int(x) for x in recv_counts.tolist()]
    recv = t.empty((sum(recv_splits), 4), dtype=send.dtype, device=send.device)
    yield ("alltoallv", recv, send, recv_splits, send_splits)
    # 4. fused pass on the owned points; partials + owned-voxel mass reduced in one call
    res = ops.fuse(recv, lo_hi)
    red = t.cat([res.partials.reshape(-1), res.mass.reshape(-1)]).to(t.float64)
    yield ("allreduce", red, "sum")
    # 5. per-point results back to the ranks the points came from
    rows = ops.pack_results(res)
    back = t.empty((n, rows.shape[1]), dtype=rows.dtype, device=rows.device)
    yield ("alltoallv", back, rows, send_splits, recv_splits)
    out = ops.unpack_results(back, send, n, p, nwords)
    return ShardedResult(out, red[: k + 6], red[k + 6 :], lo_hi, k, sum(recv_splits))


def padded_capacity(n_local: int, world: int, slack: float = 1.25) -> int:
    """Rows per peer block of the fixed-capacity exchange: this rank's share for one owner with
    slack (the global cuts balance owners; a rank's points spread over them unless its input
    range is spatially sorted — then the exchange flags an overflow and the caller re-runs)."""
    return max(64, int(slack * n_local / max(1, world)) + 64)


def cell_sharded_steps_padded(points, rank: int, world: int, ops, *, k: int, p: int, nwords: int,
                              capacity: int, lo_hi=None):
    """The cell-range protocol with a fixed-capacity exchange: every collective has host-known
    sizes and nothing is read back to the host, so the whole step can be captured in a CUDA graph.
    `capacity` rows per peer block (padded_capacity); `lo_hi` (6,) f64 device tensor = a fixed voxel
    domain shared by all ranks (drops the bbox all-reduce), None = the union of the ranks' bboxes.
    Every rank runs the fused pass on world * capacity points (NaN padding slots are inert)."""
    import torch as t

    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    n = int(points.shape[0])
    # 1. shared voxel domain (skipped for a fixed domain)
    if lo_hi is None:
        lo_hi = ops.bbox(points)
        lo_hi[3:].neg_()
        yield ("allreduce", lo_hi, "min")
        lo_hi[3:].neg_()
    # 2. cell keys + global histogram -> identical cuts on every rank
    keys, hist = ops.keys(points, lo_hi)
    yield ("allreduce", hist, "sum")
    cuts = ops.cuts(hist, world)
    # 3. points to their owners: equal-split all-to-all of fixed blocks, counts in-band
    send, flags = ops.pack_padded(points, keys, cuts, world, capacity)
    recv = t.empty_like(send)
    yield ("alltoall", recv, send)
    xyz = ops.unpad(recv, world, capacity)
    # 4. fused pass on world * capacity slots; partials + owned-voxel mass + the overflow flag in one
    #    reduction (the flag as a double: any rank's dropped points make the sum > 0)
    res = ops.fuse_points(xyz, lo_hi)
    red = t.cat([res.partials.reshape(-1), res.mass.reshape(-1), flags.to(t.float64)]).to(t.float64)
    yield ("allreduce", red, "sum")
    # 5. result rows back in slot order, equal splits
    rows = ops.pack_results(res).reshape(world, capacity, -1)
    back = t.empty_like(rows)
    yield ("alltoall", back, rows)
    out = ops.unpack_results_padded(back.reshape(world * capacity, -1), send, n, p, nwords, world, capacity)
    received = res.counts.shape[0]  # slots (device-side count of real points: (codes >= 0).sum())
    return ShardedResult(out, red[: k + 6], red[k + 6 : k + 8], lo_hi, k, received, overflow=red[k + 8])


def run_dist(gen, group=None):
    """Drive one rank's generator with torch.distributed collectives."""
    import torch.distributed as dist

    try:
        req = next(gen)
        while True:
            kind = req[0]
            if kind == "allreduce":
                op = dist.ReduceOp.SUM if req[2] == "sum" else dist.ReduceOp.MIN
                dist.all_reduce(req[1], op=op, group=group)
            elif kind == "alltoall":
                dist.all_to_all_single(req[1], req[2], group=group)
            elif kind == "alltoallv":
                _, recv, send, rs, ss = req
                dist.all_to_all_single(recv, send, output_split_sizes=rs, input_split_sizes=ss, group=group)
            else:
                raise ValueError(f"unknown collective {kind}")
            req = gen.send(None)
    except StopIteration as stop:
        return stop.value


def run_loopback(gens):
    """Drive W virtual ranks' generators in lockstep in one process; returns their results."""
    import torch as t

    world = len(gens)
    reqs, done = [], [None] * world
    for g in gens:
        reqs.append(next(g))
    while True:
        kinds = {r[0] for r in reqs}
        if len(kinds) != 1:
            raise RuntimeError(f"ranks disagree on the next collective: {kinds}")
        kind = reqs[0][0]
        if kind == "allreduce":
            stacked = t.stack([r[1] for r in reqs])
            red = stacked.sum(0) if reqs[0][2] == "sum" else stacked.amin(0)
            for r in reqs:
                r[1].copy_(red.to(r[1].dtype))
        elif kind == "alltoall":
            for dst in range(world):
                for src in range(world):
                    reqs[dst][1][src] = reqs[src][2][dst]
        elif kind == "alltoallv":
            offs = []
            for src in range(world):
                ss = reqs[src][4]
                offs.append([sum(ss[:q]) for q in range(world)])
            for dst in range(world):
                parts = [reqs[src][2][offs[src][dst] : offs[src][dst] + reqs[src][4][dst]] for src in range(world)]
                if reqs[dst][1].shape[0]:
                    reqs[dst][1].copy_(t.cat(parts))
        else:
            raise ValueError(f"unknown collective {kind}")
        nxt = []
        for q, g in enumerate(gens):
            try:
                nxt.append(g.send(None))
            except StopIteration as stop:
                done[q] = stop.value
                nxt.append(None)
        if all(x is None for x in nxt):
            return done
        if any(x is None for x in nxt):
            raise RuntimeError("ranks finished at different steps")
        reqs = nxt


def cell_sharded_fuse(points, views, tables, *, rank=None, world=None, group=None, temperature=0.1,
                      epsilon=0.01, grid=64, ops=None):
    """One rank's call (torch.distributed initialised): this rank's points (any subset of the
    object, e.g. its shard_range) -> ShardedResult with global mass/partials."""
    import torch.distributed as dist

    rank = dist.get_rank(group) if rank is None else rank
    world = dist.get_world_size(group) if world is None else world
    ops = ops or DeviceShardOps(views, tables, temperature=temperature, epsilon=epsilon, grid=grid)
    gen = cell_sharded_steps(points, rank, world, ops, k=tables.k, p=tables.p, nwords=(views.nviews + 31) // 32)
    return run_dist(gen, group)
