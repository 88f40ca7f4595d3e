"""Waveform text output: the native multi-threaded
formatter (emt_waves_to_text) against the reference's own WaveformSet::to_text
(proj/src/waveform.cpp:22-42, via oracle/_ref) and printf "%.17g"."""
import numpy as np
import pytest

from oracle import ref
from paper_1903_01081_b200 import engine

SPECIAL = [0.0, -0.0, 1.0, -1.0, 0.1, 1e-300, 5e-324, -5e-324, 1.7976931348623157e308, 1e16, 1e17, 123456789012345678.0,
           1e-5, 1e-4, 0.5, 2.0 / 3.0, float("inf"), float("-inf"), 1e21, 1e22, 9.999999999999999e22]


def _values(rows, cols, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((rows, cols)) * 10.0 ** rng.integers(-30, 30, size=(rows, cols))
    flat = v.reshape(-1)
    flat[: len(SPECIAL)] = SPECIAL[: flat.size]
    return v


def _printf(channels, width, time, values):
    head = ["time"]
    for c in channels:
        head += [c] if width == 1 else [f"{c}#{l}" for l in range(width)]
    rows = [" ".join(["%.17g" % time[r]] + ["%.17g" % x for x in values[r]]) for r in range(len(time))]
    return "\n".join([" ".join(head)] + rows) + "\n"


@pytest.mark.parametrize("width,threads", [(1, 1), (3, 4), (5, 16)])
def test_matches_printf(width, threads):
    ch = ["v(bus1)", "i(sw00)"]
    rows = 257
    t = (np.arange(rows) + 1) * 5e-5
    v = _values(rows, len(ch) * width, 7 + width)
    got = engine.waves_to_text(ch, width, t, v, threads).decode()
    assert got == _printf(ch, width, t, v)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("width", [1, 4])
def test_matches_reference_to_text(width):
    ch = ["a", "b", "c"]
    rows = 129
    t = (np.arange(rows) + 1) * 5e-5
    v = _values(rows, len(ch) * width, 11 + width)
    v[1, 0], v[1, 1] = np.nan, -np.nan  # printf spells these "nan" / "-nan"
    assert engine.waves_to_text(ch, width, t, v, 8).decode() == ref.waves_text(ch, width, t, v)


def test_empty_and_waveformset():
    assert engine.waves_to_text(["x"], 2, np.zeros(0), np.zeros((0, 2))).decode() == "time x#0 x#1\n"
    w = engine.WaveformSet(["p"], 1, np.array([5e-5, 1e-4]), np.array([[1.5], [-0.0]]))
    assert w.to_text() == "time p\n5.0000000000000002e-05 1.5\n0.0001 -0\n"
