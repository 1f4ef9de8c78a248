"""Small fused-path invocations for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py mini_bf16

Cases: `mini` (f32, SIMT kernel), `mini_bf16` (bf16, D=256: the tcgen05 tile path
k_tile_prep + k_tile_ws + sub-tiles + SIMT overflow), `pr1` (f32 SIMT at the PR1 shape) and `x3_70k`
(f32 maps, 70k points: the x3 tile path with hi/lo operand splits). Each case runs the fused call
twice on reused buffers (the second pass exercises the voxel re-zeroing), checks the status word,
and compares counts / codes against the first pass. Exits non-zero on any mismatch.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2511_03126_b200 as pf  # noqa: E402
from paper_2511_03126_b200 import workloads  # noqa: E402

CASES = {
    "mini": ("mini", None),
    "mini_bf16": ("mini_bf16", None),
    "pr1": ("pr1", None),
    "x3_70k": ("c2", 70_000),
}


def run(case: str) -> None:
    import torch

    name, n = CASES[case]
    wl = workloads.generate(name, n=n)
    views = pf.ViewSet.from_views(wl.views())
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    pts = torch.from_numpy(wl.points).cuda()
    kw = dict(temperature=wl.cfg.temperature, epsilon=wl.cfg.eps, grid=wl.cfg.grid)
    r1 = pf.fuse_and_query(pts, views, tables, check=True, **kw)
    c1, k1, m1 = r1.counts.clone(), r1.codes.clone(), r1.mass_kg()
    r2 = pf.fuse_and_query(pts, views, tables, buffers=r1.buffers, check=True, **kw)
    torch.cuda.synchronize()
    assert torch.equal(c1, r2.counts) and torch.equal(k1, r2.codes), f"{case}: rerun differs"
    assert abs(r2.mass_kg() - m1) <= 1e-6 * abs(m1), f"{case}: mass {m1} vs {r2.mass_kg()}"
    print(f"{case}: n={wl.cfg.n if n is None else n} mass={m1:.6f} ok", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        run(c)
