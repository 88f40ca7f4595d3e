"""Bergeron line extension (BASELINE C4): analytic checks of the oracle's line
model, the line-split == unsplit equivalence, and (GPU) engine == oracle.

The reference has no line model, so this parity is "unpinned"
against the reference: the closed forms below (lossless line, DC step, flat
start) are the pin. Rows r of a waveform are times t_{r+1} (proj/src/exec.cpp:366).
"""
import gzip
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bitwise_equal, within_tolerance
from oracle import oracle
from paper_1903_01081_b200 import lines
from paper_1903_01081_b200 import schedule as sch

E, ZC, RS, DT = 1000.0, 400.0, 400.0, 50e-6


def line_case(name, tau, width=1, spec=None):
    d = os.path.join(GOLDEN, "lines")
    s = gzip.open(os.path.join(d, f"{name}.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(d, f"{name}.state.gz"), "rt").read())
    ids = json.load(open(os.path.join(d, f"{name}.json")))["component_ids"]
    spec = spec or lines.single_line_spec(ZC, tau, width)
    return lines.bergeron_batch(s, st, ids, spec)


def run_oracle(batch, steps):
    return oracle.Schedule(batch.text()).interpret(batch.initial, steps)


def cols(batch, lane=0):
    """(v_a, v_b) column indices of `lane`."""
    return 0 * batch.width + lane, 1 * batch.width + lane


def test_open_end_doubles_after_one_travel_time():
    K = 10
    b = line_case("line_open", K * DT)
    w = run_oracle(b, 6 * K).waves
    ca, cb = cols(b)
    np.testing.assert_allclose(w[:K, cb], 0.0, atol=1e-12)           # wave not yet arrived
    np.testing.assert_allclose(w[K:, cb], E, rtol=1e-12)            # open end: 2 x incident E/2
    np.testing.assert_allclose(w[:2 * K, ca], E / 2, rtol=1e-12)    # incident wave E/2 (rs = Zc)
    np.testing.assert_allclose(w[2 * K:, ca], E, rtol=1e-12)        # reflection back after 2 tau


def test_matched_load_absorbs():
    K = 7
    b = line_case("line_matched", K * DT)
    w = run_oracle(b, 8 * K).waves
    ca, cb = cols(b)
    np.testing.assert_allclose(w[:, ca], E / 2, rtol=1e-12)         # no reflection ever returns
    np.testing.assert_allclose(w[:K, cb], 0.0, atol=1e-12)
    np.testing.assert_allclose(w[K:, cb], E / 2, rtol=1e-12)


def test_fractional_travel_time_interpolates():
    K, f = 10, 0.4
    b = line_case("line_open", (K + f) * DT)
    w = run_oracle(b, 4 * K).waves
    _, cb = cols(b)
    np.testing.assert_allclose(w[:K, cb], 0.0, atol=1e-12)
    np.testing.assert_allclose(w[K, cb], E * (1.0 - f), rtol=1e-12)  # linear history interpolation
    np.testing.assert_allclose(w[K + 1:2 * K, cb], E, rtol=1e-12)


def test_line_split_across_lanes_equals_unsplit():
    """A line whose ends sit in two different lanes (decoupled nodal systems, the C4
    split) gives bit-identical waveforms to the same line inside one lane."""
    tau = 6.6 * DT
    one = run_oracle(line_case("line_open", tau), 300).waves
    peers = np.array([[(1, 1), (1, 0)], [(0, 1), (0, 0)]])  # lane0.a <-> lane1.b, lane1.a <-> lane0.b
    spec = lines.LineSpec(["la", "lb"], [ZC, ZC], [tau, tau], peers)
    two = line_case("line_open", tau, spec=spec)
    w = run_oracle(two, 300).waves
    assert bitwise_equal(w[:, 0], one[:, 0]) and bitwise_equal(w[:, 3], one[:, 1])  # lane0 v_a, lane1 v_b
    assert bitwise_equal(w[:, 1], one[:, 0]) and bitwise_equal(w[:, 2], one[:, 1])


def test_spec_validation():
    spec = lines.c4_spec(8)
    lines.check_symmetric(spec)
    bad = lines.c4_spec(8)
    bad.peers[3, 2] = (0, 2)
    with pytest.raises(ValueError):
        lines.check_symmetric(bad)
    with pytest.raises(ValueError):
        line_case("line_open", 1.5 * DT)  # K < 2


def c4_case(copies):
    import bench
    s, st, ids = bench.load_case("ieee39_c4")
    return lines.c4_batch(s, st, ids, copies)


def test_c4_oracle_runs_and_lines_carry_power():
    b = c4_case(4)
    r = run_oracle(b, 600)
    assert np.all(np.isfinite(r.waves))
    i_cols = [3 * b.width + l for l in range(b.width)]  # i:pa_h
    assert np.abs(r.waves[100:, i_cols]).max() > 1.0


# ------------------------------------------------------------------ GPU parity

@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["auto", "generic", "tsimt"])
@pytest.mark.parametrize("name,tau", [("line_open", 10 * DT), ("line_open", 6.6 * DT), ("line_matched", 3 * DT)])
def test_engine_line_bitwise_equals_oracle(name, tau, kernel):
    from paper_1903_01081_b200 import engine
    k = {"auto": engine.KERNEL_AUTO, "generic": engine.KERNEL_GENERIC, "tsimt": engine.KERNEL_TSIMT}[kernel]
    b = line_case(name, tau)
    want = run_oracle(b, 400)
    eng = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, kernel=k)
    eng.reserve(400)
    eng.advance(400)
    assert bitwise_equal(eng.waves().values, want.waves)
    assert bitwise_equal(eng.state()[: b.initial.size], want.final_arena)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["auto", "generic", "tsimt"])
def test_engine_c4_matches_oracle(kernel):
    """C4 line-split batch (cross-lane, cross-CTA ring reads; launches capped at K-1 passes)."""
    from paper_1903_01081_b200 import engine
    k = {"auto": engine.KERNEL_AUTO, "generic": engine.KERNEL_GENERIC, "tsimt": engine.KERNEL_TSIMT}[kernel]
    b = c4_case(40)  # 2 CTAs of 32 lanes for the specialised kernel
    want = run_oracle(b, 900)
    eng = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, kernel=k)
    eng.reserve(900)
    eng.advance(900)
    assert within_tolerance(eng.waves().values, want.waves)
    st = eng.stats()
    if kernel == "auto":  # specialised kernel: one persistent launch (+ its source table), CTAs synchronised by progress words
        assert st.kernel_launches <= 2, eng.summary
    else:                 # launches of K-1 = 5 passes, ordered by the kernel boundary
        assert st.kernel_launches >= 900 // 5


@pytest.mark.gpu
def test_engine_c4_kernels_agree_bitwise():
    from paper_1903_01081_b200 import engine
    b = c4_case(40)
    out = []
    for k in (engine.KERNEL_SPECIALISED, engine.KERNEL_GENERIC, engine.KERNEL_TSIMT):
        eng = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, kernel=k)
        eng.reserve(700)
        eng.advance(700)
        out.append(eng.waves().values)
    assert bitwise_equal(out[0], out[1]) and bitwise_equal(out[0], out[2])


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["auto", "generic", "tsimt"])
def test_line_split_shards_with_ring_exchange_equal_one_engine(kernel):
    """Two lane-shard engines (the 2-GPU split, here on one device) that swap
    their mirror rows after every launch of K-1 passes == one engine on all lanes."""
    import torch
    from paper_1903_01081_b200 import engine
    k = {"auto": engine.KERNEL_AUTO, "generic": engine.KERNEL_GENERIC, "tsimt": engine.KERNEL_TSIMT}[kernel]
    b = c4_case(40)
    whole = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, kernel=k)
    whole.reserve(600)
    whole.advance(600)
    want = whole.waves().values
    shards, mirrors = [], []
    for lo, hi in ((0, 24), (24, 40)):
        e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, kernel=k,
                          lane_begin=lo, lane_count=hi - lo)
        ptr, lanes, cols, mc = e.ring()
        assert ptr and lanes == 40 and mc == 5
        m = torch.zeros((lanes, cols), dtype=torch.float64, device="cuda")
        e.attach_ring(m.data_ptr())
        e.reserve(600)
        shards.append((e, lo, hi))
        mirrors.append(m)
    done = 0
    while done < 600:
        n = min(5, 600 - done)
        for e, _, _ in shards:
            e.advance(n)
        for e, _, _ in shards:
            e.sync()
        torch.cuda.synchronize()
        mirrors[1][0:24] = mirrors[0][0:24]
        mirrors[0][24:40] = mirrors[1][24:40]
        torch.cuda.synchronize()
        done += n
    for (e, lo, hi) in shards:
        got = e.waves().values
        nch = len(e.channel_names)
        for c in range(nch):
            assert bitwise_equal(got[:, c * (hi - lo):(c + 1) * (hi - lo)], want[:, c * 40 + lo:c * 40 + hi])


@pytest.mark.gpu
@pytest.mark.parametrize("system_scope", [False, True])
def test_line_split_device_exchange_equals_one_engine(system_scope):
    """Two lane-shard engines sharing one mirror + progress array (the multi-GPU layout,
    here both on one device) run concurrently with no host exchange == one engine."""
    import torch
    from paper_1903_01081_b200 import engine
    b = c4_case(40)
    whole = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
    whole.reserve(700)
    whole.advance(700)
    want = whole.waves().values
    shards = []
    for lo, hi in ((0, 24), (24, 40)):
        e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, lane_begin=lo,
                          lane_count=hi - lo)
        shards.append((e, lo, hi))
    _, lanes, cols, _ = shards[0][0].ring()
    mirror = torch.zeros((lanes, cols), dtype=torch.float64, device="cuda")
    progress = torch.zeros(2, dtype=torch.int32, device="cuda")
    for k, (e, lo, hi) in enumerate(shards):
        e.attach_lines(mirror.data_ptr(), progress.data_ptr(), k, 2, system_scope)
        e.reserve(700)
    torch.cuda.synchronize()
    for e, _, _ in shards:
        e.advance(350)  # both launches in flight together, synchronised by the progress words
    for e, _, _ in shards:
        e.advance(350)
    for e, _, _ in shards:
        e.sync()
    for e, lo, hi in shards:
        got = e.waves().values
        for c in range(len(e.channel_names)):
            assert bitwise_equal(got[:, c * (hi - lo):(c + 1) * (hi - lo)], want[:, c * 40 + lo:c * 40 + hi])
        assert e.stats().kernel_launches <= 4


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["device", "host"])
def test_line_split_two_processes_bitwise(mode):
    """Two ranks (torchrun, sharing the one GPU) run a C4 shard each — device mode over a
    CUDA-IPC mirror + progress array, host mode with all-gathers — and reload once;
    rank 0 compares both runs with a single engine bit for bit (tools/linesplit_check.py)."""
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, BENCH_SHARE_GPU="1")
    root = os.path.dirname(GOLDEN.rstrip("/")).rsplit("/tests", 1)[0]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), "tools/linesplit_check.py", mode],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("linesplit") and "bitwise" in l]
    assert lines and "bitwise OK" in lines[-1], out.stdout[-2000:] + out.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["auto", "generic", "system"])
def test_document_declared_line_on_device(kernel):
    """A document with a `transmission_line` component (tests/golden/lines/line_doc.document.json,
    compiled by tools/make_line_doc_fixture.py) runs bit-identically to the C oracle."""
    from paper_1903_01081_b200 import engine
    d = os.path.join(GOLDEN, "lines")
    s = gzip.open(os.path.join(d, "line_doc.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(d, "line_doc.state.gz"), "rt").read())
    k = {"auto": engine.KERNEL_AUTO, "generic": engine.KERNEL_GENERIC, "system": engine.KERNEL_SYSTEM}[kernel]
    got = engine.interpret(s, st, 400, kernel=k)
    want = oracle.Schedule(s).interpret(st, 400)
    assert bitwise_equal(got.values, want.waves)
    assert np.abs(want.waves[:, 1]).max() > 0.0  # the wave reached the far bus
