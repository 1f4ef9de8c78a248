"""The torch.distributed NCCL branch of `dist.run_dist` (only gloo and the
loopback driver had executed it). One process, one rank, NCCL over the test box's GPU: both the
variable-size cell-range protocol and the fixed-capacity padded one run their collectives through
NCCL (all-reduce, all-to-all) and must reproduce the single-GPU call exactly. Runs in a subprocess so
the NCCL process group never touches the pytest process."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_2511_03126_b200 as pf
from paper_2511_03126_b200 import dist as pdist, workloads

torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=0, world_size=1)
try:
    for name in ("mini", "mini_bf16"):
        wl = workloads.generate(name)
        views = pf.ViewSet.from_views(wl.views())
        tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0)
        pts = torch.from_numpy(np.ascontiguousarray(wl.points)).cuda()
        one = pf.fuse_and_query(pts, views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps,
                                grid=wl.cfg.grid, check=True)
        ops = pdist.DeviceShardOps(views, tables, temperature=wl.cfg.temperature, epsilon=wl.cfg.eps,
                                   grid=wl.cfg.grid)
        nw = (views.nviews + 31) // 32
        var = pdist.run_dist(pdist.cell_sharded_steps(pts, 0, 1, ops, k=tables.k, p=tables.p, nwords=nw))
        cap = pdist.padded_capacity(pts.shape[0], 1)
        pad = pdist.run_dist(pdist.cell_sharded_steps_padded(pts, 0, 1, ops, k=tables.k, p=tables.p, nwords=nw,
                                                             capacity=cap))
        torch.cuda.synchronize()
        for r in (var, pad):
            assert torch.equal(r.counts, one.counts), name
            assert torch.equal(r.codes, one.codes), name
            assert torch.equal(r.mask_bits, one.mask_bits), name
            tol = 1e-2 if wl.cfg.bf16 else 1e-4
            assert abs(r.mass_kg() - one.mass_kg()) <= tol * abs(one.mass_kg()), (name, r.mass_kg(), one.mass_kg())
        assert not pad.overflowed()
    print("NCCL-OK")
finally:
    dist.destroy_process_group()
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_run_dist_over_nccl_one_rank(cuda):
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(_port())], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "NCCL-OK" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
