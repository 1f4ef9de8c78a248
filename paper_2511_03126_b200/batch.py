"""Batched throughput over many independent objects (BASELINE config 4; SURVEY §8e "config 4 shards
object-wise").

The reference runs one capture per `run_pipeline` call (pipeline.py:154, 224-312). A batch here is
B objects, each with its own points, views and material tables, processed by `fuse_batch` with:

* packed outputs: per-point rows of all objects back to back (`offsets[i]:offsets[i+1]`), one
  (B, 2) mass tensor and one (B, K+6) partials tensor — no per-object allocation;
* `streams` CUDA streams, objects dealt round-robin, each stream with its own workspace + voxel
  grid (sequential reuse on a stream is safe), so one object's G-table build, kernel tail and
  voxel-mass reduction overlap another's fused pass;
* multi-GPU: objects are range-sharded across ranks (`dist.shard_range(B, rank, world)`) with no
  collective — replica-style, as SURVEY §8e prescribes for config 4.

    res = fuse_batch(points_list, views_list, tables_list, temperature=0.1, epsilon=0.01, grid=128)
    res.props[res.offsets[i]:res.offsets[i + 1]]   # object i's (n_i, P) properties
    res.mass[i, 0]                                  # object i's voxel-grid mass (kg)
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .device import require_cuda, stream_handle, torch
from .errors import BundleStructureError
from .fused import FuseBuffers, _make_args


@dataclass
class BatchResult:
    offsets: list          # B + 1 row offsets into the packed per-point outputs
    props: object          # (sum N, P) f32
    counts: object         # (sum N,) i32
    codes: object          # (sum N,) i32
    mask_bits: object      # (sum N, ceil(V/32)) i32 (V = max views of the batch)
    mass: object           # (B, 2) f64 {mass_kg, occupied voxels}
    partials: object       # (B, K + 6) f64 (pf_fuse_query partial layout)
    status: object         # (B,) i32 (bit 0: NaN similarity)

    def object_props(self, i: int):
        return self.props[self.offsets[i] : self.offsets[i + 1]]


class BatchWorkspace:
    """Per-stream scratch (workspace, voxel grid, touched-voxel list) sized for the largest object
    of a batch; reusable across batches of the same shapes."""

    def __init__(self, max_n, views, tables, grid, streams, device, ws_bytes=0):
        t = torch()
        self.max_n, self.grid, self.device = int(max_n), int(grid), device
        self.bufs = [FuseBuffers(max_n, views, tables, grid, device=device) for _ in range(streams)]
        for wb in self.bufs:
            if wb.workspace.numel() < ws_bytes:
                wb.workspace = t.empty(int(ws_bytes), dtype=t.uint8, device=device)
        self.ws_bytes = min(int(wb.workspace.numel()) for wb in self.bufs)
        self.streams = [t.cuda.Stream(device=device) for _ in range(streams)]

    def fits(self, max_n, grid, streams, ws_bytes):
        return (max_n <= self.max_n and grid == self.grid and streams == len(self.streams)
                and ws_bytes <= self.ws_bytes)


def fuse_batch(points_list, views_list, tables_list, *, temperature: float = 0.1, epsilon: float = 0.01,
               grid: int = 64, streams: int = 2, workspace: BatchWorkspace | None = None):
    """Run the fused path over B objects; returns (BatchResult, BatchWorkspace). Every object's
    views / tables must share the batch's D, K and P (the packed outputs are uniform)."""
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    b = len(points_list)
    if not (len(views_list) == len(tables_list) == b) or b == 0:
        raise BundleStructureError("fuse_batch needs B >= 1 points / views / tables entries")
    dev = require_cuda()
    t = torch()
    ks = {tb.k for tb in tables_list}
    ps = {tb.p for tb in tables_list}
    if len(ks) != 1 or len(ps) != 1:
        raise BundleStructureError("all objects of a batch must have the same K and P")
    k, p = ks.pop(), ps.pop()
    nwords = max((v.nviews + 31) // 32 for v in views_list)
    pts = []
    for x in points_list:
        if hasattr(x, "is_cuda") and x.is_cuda and x.dtype == t.float32 and x.is_contiguous():
            pts.append(x.reshape(-1, 3))
        else:
            from .device import to_dev

            pts.append(to_dev(x, t.float32, dev).reshape(-1, 3))
    sizes = [int(x.shape[0]) for x in pts]
    offsets = [0]
    for s in sizes:
        offsets.append(offsets[-1] + s)
    total = offsets[-1]
    res = BatchResult(offsets=offsets,
                      props=t.empty((total, p), dtype=t.float32, device=dev),
                      counts=t.empty(total, dtype=t.int32, device=dev),
                      codes=t.empty(total, dtype=t.int32, device=dev),
                      mask_bits=t.zeros((total, nwords), dtype=t.int32, device=dev),
                      mass=t.zeros((b, 2), dtype=t.float64, device=dev),
                      partials=t.zeros((b, k + 6), dtype=t.float64, device=dev),
                      status=t.zeros(b, dtype=t.int32, device=dev))
    streams = max(1, min(int(streams), b))
    big = max(range(b), key=lambda i: sizes[i])
    if workspace is None:
        workspace = BatchWorkspace(sizes[big], views_list[big], tables_list[big], grid, streams, dev)
    ws_need = max(int(_lib.load().pf_fuse_workspace_bytes(
        _make_args(None, sizes[i], views_list[i], tables_list[i], temperature, epsilon, grid, workspace.bufs[0], 0)))
        for i in range(b))
    if not workspace.fits(sizes[big], grid, streams, ws_need):
        workspace = BatchWorkspace(sizes[big], views_list[big], tables_list[big], grid, streams, dev, ws_need)
    main = t.cuda.current_stream()
    start = t.cuda.Event()
    start.record(main)
    for s in workspace.streams:
        s.wait_event(start)
    for i in range(b):
        q = i % streams
        wb = workspace.bufs[q]
        with t.cuda.stream(workspace.streams[q]):
            _run_one(pts[i], sizes[i], views_list[i], tables_list[i], wb, res, i, offsets[i], nwords,
                     temperature, epsilon, grid)
    for s in workspace.streams:
        ev = t.cuda.Event()
        ev.record(s)
        main.wait_event(ev)
    return res, workspace


def _run_one(pts, n, views, tables, wb, res, i, off, nwords, temperature, epsilon, grid):
    """One object on the current stream, outputs bound to its rows of the packed batch tensors."""
    st = stream_handle()
    wb.vox_count.zero_()
    lo_hi = wb.lo_hi
    if n == 0:
        return
    _lib.call("pf_bbox", pts.data_ptr(), n, lo_hi.data_ptr(), st)
    a = _make_args(pts, n, views, tables, temperature, epsilon, grid, wb, 0)
    # bind the per-point outputs and the reductions to this object's slice of the batch tensors
    a.counts = res.counts[off : off + n].data_ptr()
    a.props = res.props[off : off + n].data_ptr()
    a.codes = res.codes[off : off + n].data_ptr()
    if views.nviews + 31 >= 32 * nwords:  # same word count: write straight into the batch rows
        a.mask_bits = res.mask_bits[off : off + n].data_ptr()
        mask_tmp = None
    else:  # fewer views than the batch's widest object: narrower rows, copied after
        w_i = (views.nviews + 31) // 32
        mask_tmp = wb.mask_bits.view(-1)[: n * w_i].view(n, w_i)
        a.mask_bits = mask_tmp.data_ptr()
    a.partials = res.partials[i].data_ptr()
    a.status = res.status[i : i + 1].data_ptr()
    _lib.call("pf_fuse_query", a, st)
    if mask_tmp is not None:
        res.mask_bits[off : off + n, : mask_tmp.shape[1]].copy_(mask_tmp)
    _lib.call("pf_voxel_mass_sparse", wb.grid_partials.data_ptr(), grid, wb.vox_list.data_ptr(),
              wb.vox_count.data_ptr(), n, lo_hi.data_ptr(), res.mass[i].data_ptr(), st)
