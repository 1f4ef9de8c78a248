import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))

    return load


_WL = {}


@pytest.fixture(scope="session")
def workload():
    from paper_2511_03126_b200 import workloads

    def get(name, **kw):
        key = (name, tuple(sorted(kw.items())))
        if key not in _WL:
            _WL[key] = workloads.generate(name, **kw)
        return _WL[key]

    return get


@pytest.fixture(scope="session")
def cuda():
    """Skip-free guard: gpu-marked tests must FAIL (not skip) without a GPU."""
    import torch

    assert torch.cuda.is_available(), "gpu test run without a CUDA device"
    from paper_2511_03126_b200 import _lib

    _lib.load()
    return torch.device("cuda")
