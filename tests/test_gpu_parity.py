"""CUDA engine vs the oracle / reference goldens (runs on the B200 box: -m gpu).

Bar (north_star): waveforms within 1e-9 relative + 1e-12 absolute on every
sample; switch events, topology and factor counts bit-exact. Every case must be
bit-identical: same operation order, -fmad=false, and cos evaluated as glibc
does (csrc/libmcos.cuh), so the AC-source cases are bitwise too.
"""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, bitwise_equal, load_golden, within_tolerance
from oracle import oracle
from paper_1903_01081_b200 import engine

pytestmark = pytest.mark.gpu

KERNELS = {"auto": engine.KERNEL_AUTO, "generic": engine.KERNEL_GENERIC, "tsimt": engine.KERNEL_TSIMT,
           "system": engine.KERNEL_SYSTEM}


@pytest.mark.parametrize("kernel", sorted(KERNELS))
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_engine_matches_golden(name, kernel):
    g = load_golden(name)
    k = KERNELS[kernel]
    if g.error_code:
        with pytest.raises(engine.EmtError) as ei:
            engine.interpret(g.schedule, g.initial, g.steps, kernel=k)
        assert ei.value.status == g.error_code
        # same location as the reference: "row k" / "node index k"
        where = g.error_msg.split("|where=")[-1]
        assert where in ei.value.detail
        return
    stats = engine.ExecStats()
    w = engine.interpret(g.schedule, g.initial, g.steps, engine.ExecOptions(stats=stats), kernel=k)
    assert within_tolerance(w.values, g.waves), (name, np.max(np.abs(w.values - g.waves)))
    assert bitwise_equal(w.values, g.waves), name
    assert bitwise_equal(w.time, g.time)
    assert stats.factor_count == g.factor_count


@pytest.mark.parametrize("kernel", sorted(KERNELS))
@pytest.mark.parametrize("name", ["switched_rc", "ieee39_n1_w8", "switched_dc_w3"])
def test_switch_events_bit_exact(name, kernel):
    g = load_golden(name)
    ref_run = oracle.Schedule(g.schedule).interpret(g.initial, g.steps)
    eng = engine.Engine(g.schedule, g.initial, kernel=KERNELS[kernel])
    eng.reserve(g.steps)
    eng.advance(g.steps, sync=True)
    ev = eng.events()
    assert np.array_equal(ev, ref_run.events)
    assert eng.stats().factor_count == ref_run.factor_count


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_chunked_advance_equals_one_shot(kernel):
    g = load_golden("feeder")
    one = engine.interpret(g.schedule, g.initial, 600, kernel=KERNELS[kernel])
    eng = engine.Engine(g.schedule, g.initial, kernel=KERNELS[kernel])
    eng.reserve(600)
    for n in (1, 99, 200, 300):
        eng.advance(n)
    w = eng.waves()
    assert bitwise_equal(w.values, one.values)
    assert bitwise_equal(w.time, one.time)


@pytest.mark.parametrize("kernel", sorted(KERNELS))
@pytest.mark.parametrize("name", ["switched_dc_w3", "control_only", "rc_discharge"])
def test_final_state_matches_oracle_arena(name, kernel):
    g = load_golden(name)
    ref_run = oracle.Schedule(g.schedule).interpret(g.initial, g.steps)
    eng = engine.Engine(g.schedule, g.initial, kernel=KERNELS[kernel])
    eng.reserve(g.steps)
    eng.advance(g.steps, sync=True)
    assert bitwise_equal(eng.state(), ref_run.final_arena)


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_lane_sharding_equals_full_batch(kernel):
    g = load_golden("feeder_w4")
    full = engine.interpret(g.schedule, g.initial, 200, kernel=KERNELS[kernel])
    for begin, count in ((0, 2), (2, 2), (1, 3)):
        eng = engine.Engine(g.schedule, g.initial, lane_begin=begin, lane_count=count, kernel=KERNELS[kernel])
        eng.reserve(200)
        eng.advance(200)
        part = eng.waves()
        for j in range(count):
            assert bitwise_equal(part.lane(j).values, full.lane(begin + j).values)


def test_lanes_per_block_variants_agree():
    g = load_golden("ieee39_n1_w8")
    base = engine.interpret(g.schedule, g.initial, 400)
    for lpb in (1, 3, 8):
        eng = engine.Engine(g.schedule, g.initial, lanes_per_block=lpb, kernel=engine.KERNEL_GENERIC)
        eng.reserve(400)
        eng.advance(400)
        assert bitwise_equal(eng.waves().values, base.values)
    for warps in (1, 2, 3, 8):
        eng = engine.Engine(g.schedule, g.initial, warps=warps, kernel=engine.KERNEL_SPECIALISED)
        assert eng.kernel == engine.KERNEL_SPECIALISED
        eng.reserve(400)
        eng.advance(400)
        assert bitwise_equal(eng.waves().values, base.values), warps


@pytest.mark.parametrize("name", ["ieee39", "feeder", "ieee39_n1_w8", "cyclic_controls"])
def test_auto_selects_specialised_kernel(name):
    g = load_golden(name)
    eng = engine.Engine(g.schedule, g.initial)
    assert eng.kernel == engine.KERNEL_SPECIALISED, eng.summary
    assert "emt_cg_kernel" in eng.source


def test_specialised_equals_generic_bitwise_full_n1_sample():
    """All device kernels run the same operation order: identical bits on a 64-lane N-1 batch."""
    import bench
    batch, info = bench.build_batch(64)
    out = []
    for k in (engine.KERNEL_SPECIALISED, engine.KERNEL_GENERIC, engine.KERNEL_TSIMT):
        eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width, kernel=k)
        eng.reserve(3000)
        eng.advance(3000)
        out.append((eng.waves().values, eng.stats().factor_count, eng.events(), eng.state()))
    for other in out[1:]:
        assert bitwise_equal(out[0][0], other[0])
        assert out[0][1] == other[1]
        assert np.array_equal(out[0][2], other[2])
        assert bitwise_equal(out[0][3], other[3])


def test_shard_refactor_steps_union_is_global_factor_count():
    """Sharded engines: union of per-shard refactorisation passes == the full batch's factor_count."""
    from paper_1903_01081_b200 import sharding
    g = load_golden("ieee39_n1_w8")
    full = engine.Engine(g.schedule, g.initial)
    full.reserve(g.steps)
    full.advance(g.steps, sync=True)
    parts = []
    for r in range(3):
        lo, hi = sharding.shard_bounds(8, 3, r)
        e = engine.Engine(g.schedule, g.initial, lane_begin=lo, lane_count=hi - lo)
        e.reserve(g.steps)
        e.advance(g.steps, sync=True)
        parts.append(e.refactor_steps().tolist())
    assert sharding.combine_factor_counts(parts) == full.stats().factor_count == g.factor_count


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_load_run_streams_same_waves_as_advance(kernel):
    """emt_engine_load + emt_engine_run (chunked launches, D2H overlapped) == one-shot interpret."""
    g = load_golden("feeder_w4")
    one = engine.interpret(g.schedule, g.initial, 700, kernel=KERNELS[kernel])
    eng = engine.Engine(g.schedule, g.initial, kernel=KERNELS[kernel])
    out = np.zeros((700, eng.channels * eng.lanes))
    eng.run(700, out, chunk=64)
    assert bitwise_equal(out, one.values)
    # reload the same batch: rewinds to pass 0, same bits again; odd chunking
    eng.load(g.initial)
    out2 = np.zeros_like(out)
    eng.run(700, out2, chunk=333)
    assert bitwise_equal(out2, one.values)


def test_load_new_lane_varying_constants_equals_fresh_engine():
    """A reloaded N-1 batch with other fault times (lane-varying constants) == a fresh engine on it."""
    import bench
    from paper_1903_01081_b200 import schedule as sch
    s, st, ids = bench.load_case("ieee39")
    pick = ["sw03", "sw07", "sw19", "sw40"] * 8
    a = sch.n1_batch(s, st, ids, [(b, 0.004 + 0.0003 * k) for k, b in enumerate(pick)])
    b = sch.n1_batch(s, st, ids, [(b, 0.011 + 0.0007 * k) for k, b in enumerate(pick)])
    eng = engine.Engine(a.schedule, a.initial, const_table=a.const_table, width=a.width)
    assert eng.kernel == engine.KERNEL_SPECIALISED
    eng.load(b.initial, b.const_table)
    out = np.zeros((1200, eng.channels * eng.lanes))
    eng.run(1200, out, chunk=100)
    fresh = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
    fresh.reserve(1200)
    fresh.advance(1200)
    assert bitwise_equal(out, fresh.waves().values)
    assert np.array_equal(eng.events(), fresh.events())
    assert len(fresh.events()) == len(pick)
    assert eng.stats().factor_count == fresh.stats().factor_count


def test_load_rejects_changed_compiled_constant():
    g = load_golden("ieee39_n1_w8")
    eng = engine.Engine(g.schedule, g.initial)
    assert eng.kernel == engine.KERNEL_SPECIALISED
    ct = np.array([float(x) for ln in g.schedule.splitlines() if ln.startswith("CONST ") for x in ln.split()[2:]])
    ct = ct.reshape(-1, g.width) if ct.size % g.width == 0 else None
    if ct is None:
        pytest.skip("const table layout not row-per-slot")
    inv = [k for k in range(ct.shape[0]) if np.all(ct[k] == ct[k, 0])]
    ct2 = ct.copy()
    ct2[inv[0]] += 1.0
    with pytest.raises(engine.EmtError) as ei:
        eng.load(g.initial, ct2)
    assert ei.value.code == "TopologyMismatch"


def test_staged_batches_pipeline_equals_fresh_engines():
    """stage(next) while the current batch runs, then commit: each batch == a fresh engine on it."""
    import bench
    from paper_1903_01081_b200 import schedule as sch
    s, st, ids = bench.load_case("ieee39")
    pick = ["sw01", "sw09", "sw22", "sw37"] * 8
    batches = [sch.n1_batch(s, st, ids, [(b, t0 + 0.0005 * k) for k, b in enumerate(pick)]) for t0 in (0.003, 0.009, 0.015)]
    eng = engine.Engine(batches[0].schedule, batches[0].initial, const_table=batches[0].const_table,
                        width=batches[0].width)
    outs = []
    eng.stage(batches[0].initial, batches[0].const_table)
    for k, b in enumerate(batches):
        eng.commit()
        if k + 1 < len(batches):
            eng.stage(batches[k + 1].initial, batches[k + 1].const_table)
        out = np.zeros((900, eng.channels * eng.lanes))
        eng.run(900, out, chunk=128)
        outs.append((out, eng.events(), eng.stats().factor_count))
    for b, (out, ev, fc) in zip(batches, outs):
        fresh = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
        fresh.reserve(900)
        fresh.advance(900)
        assert bitwise_equal(out, fresh.waves().values)
        assert np.array_equal(ev, fresh.events())
        assert fc == fresh.stats().factor_count


def _pv_batch(n):
    import bench
    return bench.build_batch(n, workload="c5")[0]


def test_tensor_solve_shared_g_matches_oracle_to_amplitude_tolerance():
    """Shared-G tensor-core solve (V = G^-1 I via DMMA) reassociates the triangular
    solve: every sample within 1e-9 of its channel's amplitude (not bit-exact)."""
    b = _pv_batch(64)
    steps = 3000
    want = oracle.Schedule(b.text()).interpret(b.initial, steps)
    eng = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, tensor_solve=True)
    assert "solve=dmma" in eng.summary, eng.summary
    eng.reserve(steps)
    eng.advance(steps)
    got = eng.waves().values
    amp = np.abs(want.waves).max(axis=0)
    err = np.abs(got - want.waves)
    assert np.all(err <= 1e-9 * amp + 1e-12), float((err / (amp + 1e-300)).max())
    assert eng.stats().factor_count == want.factor_count


def test_tensor_solve_ignored_when_g_is_not_shared():
    g = load_golden("ieee39_n1_w8")  # breakers switch: G differs per lane and over time
    base = engine.interpret(g.schedule, g.initial, 600)
    eng = engine.Engine(g.schedule, g.initial, tensor_solve=True)
    assert "ineligible" in eng.summary, eng.summary
    eng.reserve(600)
    eng.advance(600)
    assert bitwise_equal(eng.waves().values, base.values)


def test_run_async_two_engines_alternating():
    """run_async/wait with two engines taking turns (the serving pipeline) == synchronous runs."""
    g = load_golden("feeder_w4")
    want = engine.interpret(g.schedule, g.initial, 500)
    engs = [engine.Engine(g.schedule, g.initial) for _ in range(2)]
    outs = [np.zeros((500, engs[0].channels * engs[0].lanes)) for _ in range(2)]
    for k in range(4):
        e = engs[k % 2]
        if k >= 2:
            e.wait()
            assert bitwise_equal(outs[k % 2], want.values)
            outs[k % 2][:] = 0.0
        e.stage(g.initial)
        e.commit()
        e.run_async(500, outs[k % 2], chunk=128)
    for k, e in enumerate(engs):
        e.wait()
        assert bitwise_equal(outs[k], want.values)


def test_fast_division_detects_subnormal_quotients_exact_mode_is_bitwise():
    """Backward-sweep quotients below 2^-900 (a decay through the subnormals): the fast
    kernel stops with InexactDivision instead of misrounding, EMT_FLAG_EXACT_DIVISION
    (IEEE fallback per row) is bit-identical to the reference, and interpret() retries
    by itself (test_engine_matches_golden covers it through the golden)."""
    g = load_golden("subnormal_decay")
    eng = engine.Engine(g.schedule, g.initial)
    assert eng.kernel == engine.KERNEL_SPECIALISED
    eng.reserve(g.steps)
    with pytest.raises(engine.EmtError) as ei:
        eng.advance(g.steps, sync=True)
    assert ei.value.code == "InexactDivision"
    ex = engine.Engine(g.schedule, g.initial, exact_division=True)
    ex.reserve(g.steps)
    ex.advance(g.steps, sync=True)
    assert bitwise_equal(ex.waves().values, g.waves)


def test_async_jit_runs_generic_then_switches_bitwise(tmp_path, monkeypatch):
    """EMT_FLAG_ASYNC_JIT: creation returns at once, the generic kernel runs while the
    specialised one compiles on a host thread (empty cubin cache here), and the switch
    at a launch boundary leaves every sample bit-identical to a synchronous run."""
    import bench
    monkeypatch.setenv("EMTB200_CACHE", str(tmp_path))
    batch, _ = bench.build_batch(48)  # a width no other test compiles: no in-memory cache hit
    steps = 1200
    eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width,
                        async_jit=True)
    eng.reserve(steps)
    eng.advance(100)
    eng.advance(100)
    first = eng.kernel
    eng.wait_jit()
    eng.advance(steps - 200)
    assert eng.kernel == engine.KERNEL_SPECIALISED, eng.summary
    assert "async JIT" in eng.summary
    assert first == engine.KERNEL_GENERIC  # NVRTC takes seconds: the first launches ran generic
    ref = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width)
    ref.reserve(steps)
    ref.advance(steps)
    assert bitwise_equal(eng.waves().values, ref.waves().values)
    assert np.array_equal(eng.events(), ref.events())
    assert eng.stats().factor_count == ref.stats().factor_count
    assert bitwise_equal(eng.state(), ref.state())


def test_async_jit_engine_closed_while_compiling_and_serving_paths(tmp_path, monkeypatch):
    """Destroying an engine whose JIT is still compiling waits for the host thread; the
    staged-batch serving path (stage / commit / run_async) across the switch stays bitwise."""
    import bench
    monkeypatch.setenv("EMTB200_CACHE", str(tmp_path))
    batch, _ = bench.build_batch(40)
    e = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width, async_jit=True)
    e.close()  # compile still in flight: the destructor joins it
    ref = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width)
    ref.reserve(600)
    ref.advance(600)
    want = ref.waves().values
    e = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width, async_jit=True)
    outs = []
    for k in range(3):
        e.stage(batch.initial, batch.const_table)
        e.commit()
        out = np.zeros((600, e.channels * e.lanes))
        e.run_async(600, out, chunk=100)
        e.wait()
        outs.append(out)
        if k == 0:
            e.wait_jit()
    assert e.kernel == engine.KERNEL_SPECIALISED
    for out in outs:
        assert bitwise_equal(out, want)


@pytest.mark.parametrize("name,devices", [("ieee39_n1_w8", (0, 0, 0)), ("feeder_w4", (0, 0)), ("switched_dc_w3", (0,))])
def test_multi_device_executor_equals_interpret(name, devices):
    """emt_create / emt_run: lane shards over the listed devices (one
    device listed several times here), waves in the batch layout and the batch's
    factor_count (a pass counts once when any lane refactorises), bitwise."""
    g = load_golden(name)
    w, st = engine.run_devices(g.schedule, g.initial, g.steps, devices=devices, warmup=10)
    assert bitwise_equal(w.values, g.waves)
    assert bitwise_equal(w.time, g.time)
    assert st.factor_count == g.factor_count
    assert st.measured_steps == g.steps - 10


def test_multi_device_executor_reports_errors():
    g = load_golden("singular_islands")
    with pytest.raises(engine.EmtError) as ei:
        engine.run_devices(g.schedule, g.initial, g.steps, devices=(0, 0))
    assert ei.value.status == g.error_code


def test_execute_parallel_twin_equals_golden():
    """emt_execute_parallel: execute_parallel's contract (the reference's layer-parallel
    executor is bit-identical to interpret, exec.cpp:385); the device runs it."""
    import ctypes
    g = load_golden("ieee39_n1_w8")
    L = engine.lib()
    init = np.ascontiguousarray(g.initial)
    nch = len(engine.channel_names(g.schedule))
    waves = np.zeros((g.steps, nch * g.width))
    time = np.zeros(g.steps)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = L.emt_execute_parallel(g.schedule.encode(), init.ctypes.data_as(dp), init.size, 4, g.steps, None, None,
                                waves.ctypes.data_as(dp), time.ctypes.data_as(dp), None)
    assert rc == 0, L.emt_last_error()
    assert bitwise_equal(waves, g.waves)
    assert bitwise_equal(time, g.time)


def test_full_chip_launch_concurrent_engines_claim_every_lane_group():
    """Full-chip launch (one CTA per SM, lane group s taken on SM s; codegen.cpp bid_code):
    three engines launched concurrently on their own streams compete for the same SMs,
    so CTAs land on SMs whose group another CTA already holds or never gets; every lane
    group must still run exactly once (CAS claims, spares take the free groups)."""
    import bench
    b, _ = bench.build_batch(96)  # three 32-lane groups of the C3 sweep (faults 0.10 s on)
    steps = 2400
    ref = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
    assert "launch=full-chip" in ref.summary, ref.summary
    ref.reserve(steps)
    ref.advance(steps, sync=True)
    want = ref.waves().values
    engs = [engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width) for _ in range(3)]
    for e in engs:
        e.reserve(steps)
    for _ in range(steps // 200):  # interleaved launches of 200 passes on three streams
        for e in engs:
            e.advance(200)
    for e in engs:
        e.sync()
        assert bitwise_equal(e.waves().values, want)
        assert len(e.events()) == len(ref.events())
