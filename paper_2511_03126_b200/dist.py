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
