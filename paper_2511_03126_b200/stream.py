"""Streaming many objects through the fused path with host transfers overlapped.

`FusePipeline` keeps two device slots (points, views, query tables, outputs) and three CUDA streams:
object i's inputs are uploaded on the H2D stream while object i-1 is computed on the compute stream
and object i-2's per-point properties come back on the D2H stream. Every object still pays its own
uploads and downloads — they only stop serialising with the compute. This is the serving form of
`fuse_and_query` (the reference processes one capture per `run_pipeline` call, pipeline.py:154).

    pipe = FusePipeline(n, nviews, image_hw, fmap_shape, bf16=True, k=K, p=2, grid=512)
    for res in pipe.run(objects):          # HostObject items, pinned host tensors
        res.props                          # (n, P) host tensor, valid until the next result is requested
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import ViewSet, require_cuda, torch
from .fused import FuseBuffers, QueryTables, fuse_and_query


@dataclass
class HostObject:
    """One capture on the host (pinned tensors for overlapped copies)."""

    points: object      # (N, 3) f32
    rotation: np.ndarray  # (V, 3, 3) f64 world->camera (bundle.py:35-56)
    translation: np.ndarray  # (V, 3) f64
    intrinsics: np.ndarray  # (V, 4) f64 fx, fy, cx, cy
    depth: object       # (V, H, W) f32
    fmap: object        # (V, Hf, Wf, D) f32, or int16 bit patterns of bf16
    text: object        # (K, D) f32 unit rows
    values: object      # (K, P) f32
    mid_theta: object   # (K,) f32


@dataclass
class StreamResult:
    index: int
    props: object   # (N, P) host tensor
    mass: object    # (2,) host f64 tensor: voxel-grid mass (kg), occupied voxels


class FusePipeline:
    LAG = 2   # objects issued ahead of the one being yielded
    RING = 4  # host output buffers (> LAG + 1)

    def __init__(self, n: int, nviews: int, image_hw, fmap_shape, *, bf16: bool, k: int, p: int, grid: int,
                 temperature: float = 0.1, epsilon: float = 0.01, density_col: int = 0, device=None,
                 group=None, sharded: bool = False):
        """sharded=True (torch.distributed initialised): every rank streams ITS points of each
        object (e.g. its shard_range) and the objects are computed with the cell-range sharded
        path (dist.cell_sharded_steps over NCCL); `mass` is then the whole object's."""
        dev = require_cuda(device)
        t = torch()
        self.n, self.nviews, self.grid = int(n), int(nviews), int(grid)
        self.temperature, self.epsilon = float(temperature), float(epsilon)
        h, w = image_hw
        hf, wf, d = fmap_shape
        self.bf16 = bool(bf16)
        self.dev = dev
        self.slots = []
        for _ in range(2):
            pts = t.empty((n, 3), dtype=t.float32, device=dev)
            depth = t.empty((nviews, h, w), dtype=t.float32, device=dev)
            fmap = t.empty((nviews, hf, wf, d), dtype=t.bfloat16 if bf16 else t.float32, device=dev)
            eye = np.tile(np.eye(3), (nviews, 1, 1))
            views = ViewSet.from_tensors(eye, np.zeros((nviews, 3)), np.tile([1.0, 1.0, 0.0, 0.0], (nviews, 1)),
                                         depth, fmap, device=dev)
            tables = QueryTables.build(np.zeros((k, d), np.float32), np.zeros((k, p), np.float32),
                                       np.zeros(k, np.float32), density_col=density_col, device=dev)
            bufs = None if sharded else FuseBuffers(n, views, tables, grid, device=dev)
            rec_pinned = t.empty(views.records_dev.numel(), dtype=t.uint8).pin_memory()
            self.slots.append({"pts": pts, "depth": depth, "fmap": fmap, "views": views, "tables": tables,
                               "bufs": bufs, "records": rec_pinned})
        self.h2d = t.cuda.Stream(device=dev)
        self.comp = t.cuda.Stream(device=dev)
        self.d2h = t.cuda.Stream(device=dev)
        mk = lambda: t.cuda.Event()  # noqa: E731
        self.ev_h2d = [mk(), mk()]   # whole upload (the feature maps last)
        self.ev_pts = [mk(), mk()]   # records, property tables and points
        self.ev_depth = [mk(), mk()]  # + depth maps
        self.ev_comp = [mk(), mk()]
        self.ev_d2h = [mk(), mk()]
        # host output ring: a result stays valid while the next LAG objects are issued (the host never
        # blocks on a download before the following uploads and computes are queued)
        self.host_props = [t.empty((n, p), dtype=t.float32).pin_memory() for _ in range(self.RING)]
        self.host_mass = [t.empty(2, dtype=t.float64).pin_memory() for _ in range(self.RING)]
        self.h2d_bytes = 0
        self.d2h_bytes = n * p * 4 + 16
        self.sharded, self.group = bool(sharded), group
        if self.sharded:
            import torch.distributed as tdist

            from .dist import DeviceShardOps

            self.rank, self.world = tdist.get_rank(group), tdist.get_world_size(group)
            for sl in self.slots:
                sl["ops"] = DeviceShardOps(sl["views"], sl["tables"], temperature=self.temperature,
                                           epsilon=self.epsilon, grid=self.grid)

    def _upload(self, slot, obj: HostObject):
        t = torch()
        s = self.slots[slot]
        v = s["views"]
        rec = v.records
        rec["R"] = np.asarray(obj.rotation, np.float64).reshape(-1, 9)
        rec["t"] = np.asarray(obj.translation, np.float64)
        intr = np.asarray(obj.intrinsics, np.float64)
        rec["fx"], rec["fy"], rec["cx"], rec["cy"] = intr[:, 0], intr[:, 1], intr[:, 2], intr[:, 3]
        rec_host = s["records"]
        self.ev_h2d[slot].synchronize()  # the pinned record block of object i-2 has been read
        rec_host.copy_(t.from_numpy(rec.view(np.uint8).reshape(-1)))
        # staged: small tables + points (the compute starts on these), then the depth maps (first read
        # by the tile prep), then the feature maps and text (the G table and the gather)
        tb = s["tables"]
        v.records_dev.copy_(rec_host, non_blocking=True)
        tb.values.copy_(obj.values, non_blocking=True)
        tb.mid_theta.copy_(obj.mid_theta, non_blocking=True)
        s["pts"].copy_(obj.points, non_blocking=True)
        self.ev_pts[slot].record(self.h2d)
        s["depth"].view(-1).copy_(obj.depth.reshape(-1), non_blocking=True)
        self.ev_depth[slot].record(self.h2d)
        tb.text.copy_(obj.text, non_blocking=True)
        if self.bf16:
            s["fmap"].view(t.int16).view(-1).copy_(obj.fmap.reshape(-1), non_blocking=True)
        else:
            s["fmap"].view(-1).copy_(obj.fmap.reshape(-1), non_blocking=True)
        self.h2d_bytes = (obj.points.numel() * 4 + obj.depth.numel() * 4 + obj.fmap.numel() * obj.fmap.element_size()
                          + (obj.text.numel() + obj.values.numel() + obj.mid_theta.numel()) * 4 + rec_host.numel())

    def run(self, objects, events=None):
        """Generator: yields a StreamResult per object once its outputs are on the host.
        events=(start, end): CUDA events recorded before the first upload and after the last
        download (device-side timing of the whole stream)."""
        t = torch()
        pending = []
        for i, obj in enumerate(objects):
            slot = i & 1
            hb = i % self.RING
            s = self.slots[slot]
            with t.cuda.stream(self.h2d):
                if i == 0 and events is not None:
                    events[0].record(self.h2d)
                self.h2d.wait_event(self.ev_comp[slot])  # object i-2 no longer reads this slot
                self._upload(slot, obj)
                self.ev_h2d[slot].record(self.h2d)
            with t.cuda.stream(self.comp):
                # unsharded: only the points gate the start; the depth / feature-map events go into the
                # call, which waits for them where they are first read
                self.comp.wait_event(self.ev_pts[slot] if not self.sharded else self.ev_h2d[slot])
                self.comp.wait_event(self.ev_d2h[slot])  # object i-2's outputs have been downloaded
                if self.sharded:
                    from .dist import cell_sharded_steps, run_dist

                    v, tb = s["views"], s["tables"]
                    out = run_dist(cell_sharded_steps(s["pts"], self.rank, self.world, s["ops"], k=tb.k, p=tb.p,
                                                      nwords=(v.nviews + 31) // 32), self.group)
                    props_dev, mass_dev = out.props, out.mass
                    props_dev.record_stream(self.d2h)  # freed result tensors stay unreused until downloaded
                    mass_dev.record_stream(self.d2h)
                else:
                    bufs = s["bufs"]
                    bufs.reset()
                    # (the per-object G table is built inside, on a forked stream overlapping the sort)
                    fuse_and_query(s["pts"], s["views"], s["tables"], temperature=self.temperature,
                                   epsilon=self.epsilon, grid=self.grid, buffers=bufs, reset=False,
                                   depth_ready=self.ev_depth[slot], fmap_ready=self.ev_h2d[slot])
                    props_dev, mass_dev = bufs.props, bufs.mass
                self.ev_comp[slot].record(self.comp)
            with t.cuda.stream(self.d2h):
                self.d2h.wait_event(self.ev_comp[slot])
                self.host_props[hb].copy_(props_dev, non_blocking=True)
                self.host_mass[hb].copy_(mass_dev, non_blocking=True)
                self.ev_d2h[slot].record(self.d2h)
                done = t.cuda.Event()
                done.record(self.d2h)
            pending.append((i, hb, done))
            if len(pending) > self.LAG:  # yield the oldest object once its download is done
                j, h, ev = pending.pop(0)
                ev.synchronize()
                yield StreamResult(j, self.host_props[h], self.host_mass[h])
        if events is not None:
            with t.cuda.stream(self.d2h):
                events[1].record(self.d2h)
        for j, h, ev in pending:
            ev.synchronize()
            yield StreamResult(j, self.host_props[h], self.host_mass[h])
