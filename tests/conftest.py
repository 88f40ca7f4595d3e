"""Test configuration: `gpu` marks tests that need a B200 (run via gpurun)."""
import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu on the GPU box")


def read_gz(path):
    with gzip.open(path, "rt") as f:
        return f.read()


class Golden:
    def __init__(self, name):
        self.name = name
        self.schedule = read_gz(os.path.join(GOLDEN, f"{name}.cgmsched.gz"))
        self.state_text = read_gz(os.path.join(GOLDEN, f"{name}.state.gz"))
        z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
        self.waves = z["waves"]
        self.time = z["time"]
        self.factor_count = int(z["factor_count"])
        self.error_code = int(z["error_code"])
        self.error_msg = str(z["error_msg"]) if "error_msg" in z else ""
        self.meta = json.loads(str(z["meta"]))
        self.steps = self.meta["steps"]
        from paper_1903_01081_b200 import schedule as sch
        self.initial, self.width = sch.parse_state(self.state_text)


@pytest.fixture(params=GOLDEN_CASES)
def golden(request):
    return Golden(request.param)


def load_golden(name):
    return Golden(name)


def bitwise_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and bool((a.view(np.uint64) == b.view(np.uint64)).all())


def within_tolerance(a, b, rel=1e-9, abs_=1e-12):
    """north_star tolerance: |a - b| <= 1e-12 + 1e-9 |b| on every sample."""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.all(np.abs(a - b) <= abs_ + rel * np.abs(b)))
