import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name):
    from paper_1401_3615_b200.geometry import VolumeGeometry

    d = np.load(os.path.join(GOLDEN, name))
    g = VolumeGeometry(int(d["L"]), float(d["voxel_mm"]), float(d["origin_mm"]))
    return g, d["mats"], d["imgs"], d["vol0"], d["expected"]


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def cuda():
    """GPU tests fail (not skip) without a device: they are the parity gate."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    import paper_1401_3615_b200 as pkg

    assert pkg.device_count() >= 1
    return torch.device("cuda:0")
