"""The large single-system kernel (EMT_KERNEL_SYSTEM, csrc/system_kernel.cuh) on the
reference's own large-scale cases: gen_scale_case(feeder33_pv3, k) compiled by the
reference (tools/make_scale_cases.py; proj/src/bench.cpp:54-117, the paper's
large-case test), against the reference's interpret itself
(oracle/_ref/libemtref.so). Every sample bit-identical; factor counts equal.
The small goldens run through this kernel too (tests/test_gpu_parity.py, KERNELS).
"""
import numpy as np
import pytest

from conftest import bitwise_equal
from oracle import parity, ref
from paper_1903_01081_b200 import engine

pytestmark = pytest.mark.gpu


def _case(k):
    import bench
    s, st = bench.load_scale_case(k)
    return s, st


@pytest.mark.parametrize("k,steps", [(32, 4000), (128, 1500)])
def test_scale_case_bitwise_vs_reference(k, steps):
    s, st = _case(k)
    eng = engine.Engine(s, st)
    assert eng.kernel == engine.KERNEL_SYSTEM, eng.summary
    eng.reserve(steps)
    for n in (1, steps // 2 - 1, steps - steps // 2):  # launch boundaries inside the run
        eng.advance(n)
    eng.sync()
    want = ref.execute(s, st, steps)
    rep = parity.merge([parity.compare(eng.waves().values, want.waves)])
    assert rep["ok"] and rep["bitwise_fraction"] == 1.0, rep
    assert eng.stats().factor_count == want.factor_count


def test_scale_case_final_arena_and_events_vs_oracle():
    """The whole final arena (v, currents, control states, L/U, scratch) after 300 passes
    against the C oracle (pinned bit-for-bit to the reference, tests/test_oracle.py)."""
    from oracle import oracle
    s, st = _case(32)
    eng = engine.Engine(s, st, kernel=engine.KERNEL_SYSTEM)
    eng.reserve(300)
    eng.advance(300, sync=True)
    want = oracle.Schedule(s).interpret(st, 300)
    assert bitwise_equal(eng.waves().values, want.waves)
    assert bitwise_equal(eng.state(), want.final_arena)
    assert np.array_equal(eng.events(), want.events)
