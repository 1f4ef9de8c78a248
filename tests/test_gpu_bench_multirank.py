"""bench.py's N > 1 code path (cell-range sharded step + sharded FusePipeline e2e) under torchrun
with 2 ranks on the one GPU of the test box: the collectives go over gloo (PF_BENCH_BACKEND), so each
is a host-side step and no kernel waits on another rank. Timing is meaningless here; the check is
that the 2-rank job finishes and reports the same object (mass, visible pairs) as the 1-rank job."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out):
    return json.loads([x for x in out.splitlines() if x.startswith("{")][-1])


def test_two_rank_bench_matches_one_rank(cuda):
    args = ["bench.py", "--config", "pr1", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    one = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    env = dict(os.environ, PF_BENCH_DEVICE="0", PF_BENCH_BACKEND="gloo")
    # the 2-rank job takes ~15 s; one run of the suite saw the torchrun job hang (a rendezvous /
    # gloo connect on the shared host, not a kernel: every collective is a host-side step), so a
    # stuck attempt is killed and retried once on a fresh port
    two = None
    for attempt in range(2):
        try:
            two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                                  "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args, "--gpus", "2"],
                                 cwd=ROOT, capture_output=True, text=True, timeout=240, env=env)
            break
        except subprocess.TimeoutExpired as e:
            print(f"2-rank attempt {attempt} timed out; stderr tail: {(e.stderr or b'')[-1500:]!r}")
    assert two is not None, "the 2-rank job timed out twice"
    assert two.returncode == 0, two.stderr[-2000:]
    a, b = _line(one.stdout), _line(two.stdout)
    assert b["n_gpus"] == 2 and "cell-range x2" in b["config"]["parallelism"]
    assert b["result"]["visible_pairs"] == a["result"]["visible_pairs"]
    assert b["result"]["featured"] == a["result"]["featured"]
    assert b["result"]["mass_kg"] == pytest.approx(a["result"]["mass_kg"], rel=1e-5)
    assert b["e2e"]["mass_kg_last"] == pytest.approx(a["result"]["mass_kg"], rel=1e-5)
