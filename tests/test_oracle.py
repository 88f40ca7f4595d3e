"""The C restatement (oracle/emt_oracle.c) is pinned bit-for-bit to the reference.

Golden fixtures were produced by the reference library itself
(tools/make_fixtures.py -> oracle/_ref/libemtref.so -> emtgrid::interpret).
"""
import numpy as np
import pytest

from conftest import bitwise_equal, load_golden
from oracle import oracle


def test_oracle_matches_reference_golden(golden):
    s = oracle.Schedule(golden.schedule)
    if golden.error_code:
        with pytest.raises(oracle.OracleError) as ei:
            s.interpret(golden.initial, golden.steps)
        assert ei.value.code == golden.error_code
        return
    run = s.interpret(golden.initial, golden.steps)
    assert bitwise_equal(run.waves, golden.waves), golden.name
    assert bitwise_equal(run.time, golden.time)
    assert run.factor_count == golden.factor_count


def test_oracle_error_locations():
    g = load_golden("singular_islands")
    with pytest.raises(oracle.OracleError) as ei:
        oracle.Schedule(g.schedule).interpret(g.initial, g.steps)
    assert ei.value.code == 8 and ei.value.index == 1 and "row 1" in g.error_msg
    g = load_golden("diverging")
    with pytest.raises(oracle.OracleError) as ei:
        oracle.Schedule(g.schedule).interpret(g.initial, g.steps)
    assert ei.value.code == 7 and ei.value.index == 0 and ei.value.step > 0


def test_oracle_switch_events_and_factor_counts():
    g = load_golden("switched_rc")
    run = oracle.Schedule(g.schedule).interpret(g.initial, g.steps)
    # toggles at 0.3 ms and 0.6 ms with dt = 0.1 ms: t=(step+1)*dt >= t_j
    assert [tuple(e[:2]) for e in run.events] == [(2, 0), (5, 0)]
    assert run.factor_count == 3
    g = load_golden("ieee39_n1_w8")
    run = oracle.Schedule(g.schedule).interpret(g.initial, g.steps)
    assert len(run.events) == 8 and sorted(run.events[:, 1].tolist()) == list(range(8))
    assert run.factor_count == 1 + len(set(run.events[:, 0].tolist()))


def test_oracle_zero_steps_and_dimension_mismatch():
    g = load_golden("feeder")
    s = oracle.Schedule(g.schedule)
    assert s.interpret(g.initial, 0).waves.shape == (0, 5)
    with pytest.raises(oracle.OracleError) as ei:
        s.interpret(g.initial[:-1], 1)
    assert ei.value.code == 10  # DimensionMismatch


def test_oracle_rejects_unknown_kernel_code():
    g = load_golden("rc_discharge")
    lines = g.schedule.splitlines()
    k = next(i for i, ln in enumerate(lines) if ln.startswith("P "))
    f = lines[k].split()
    f[3] = "99"
    lines[k] = " ".join(f)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.Schedule("\n".join(lines) + "\n").interpret(g.initial, 1)
    assert ei.value.code == 14  # UnknownKind
