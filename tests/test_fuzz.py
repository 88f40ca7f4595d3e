"""Property-style parity: 64 seeded random documents (tests/golden/docs.py:fuzz — every
electrical kind, meshed topologies, breakers toggling several times, AC and DC
sources, a meter -> control chain -> actuator loop through all control kinds)
compiled and run by the REAL reference (tools/make_fuzz_fixtures.py). The C oracle
(CPU) and every device kernel (GPU) must reproduce the reference's waveforms bit for
bit and its refactorisation count. `fuzzw_*` are vectorised by the reference's own
override rows; `fuzzl_*` add `transmission_line` components (no reference line
model: their stored waves are the C oracle's, so they pin the device kernels)."""
import gzip
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bitwise_equal
from oracle import oracle
from paper_1903_01081_b200 import schedule as sch

FUZZ = os.path.join(GOLDEN, "fuzz")
CASES = sorted(f[:-4] for f in os.listdir(FUZZ) if f.endswith(".npz")) if os.path.isdir(FUZZ) else []


def load(name):
    s = gzip.open(os.path.join(FUZZ, f"{name}.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(FUZZ, f"{name}.state.gz"), "rt").read())
    z = np.load(os.path.join(FUZZ, f"{name}.npz"))
    return s, st, z, json.loads(str(z["meta"]))["steps"]


def test_fuzz_set_present():
    assert len(CASES) >= 78


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    s, st, z, steps = load(name)
    r = oracle.Schedule(s).interpret(st, steps)
    assert bitwise_equal(r.waves, z["waves"])
    assert r.factor_count == int(z["factor_count"])


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["auto", "generic", "tsimt", "system"])
@pytest.mark.parametrize("name", CASES)
def test_device_matches_reference(name, kernel):
    from paper_1903_01081_b200 import engine
    k = {"auto": engine.KERNEL_AUTO, "generic": engine.KERNEL_GENERIC, "tsimt": engine.KERNEL_TSIMT,
         "system": engine.KERNEL_SYSTEM}[kernel]
    s, st, z, steps = load(name)
    stats = engine.ExecStats()
    w = engine.interpret(s, st, steps, engine.ExecOptions(stats=stats), kernel=k)
    assert bitwise_equal(w.values, z["waves"]), name
    assert bitwise_equal(w.time, z["time"])
    assert stats.factor_count == int(z["factor_count"])
