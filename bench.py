#!/usr/bin/env python
"""Benchmark: IEEE-39 N-1 contingency sweep (BASELINE.json metric, config C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c5|c2|c4] [--scaling strong|weak]

Workload: the BASELINE C3 sweep — 1000 scenarios (46 breakers x 22 fault times
0.10-0.31 s, outage-major; sharding.n1_sweep) of the synthetic IEEE 39-bus EMT
case (n = 85 nodes, m = 149 components, dt = 50 us) — in contiguous lane
shards, one process per GPU under torchrun (strong scaling: 1000 scenarios in
total; `--scaling weak` runs 1000 per GPU). No inter-GPU traffic but the final
reductions / result gather. One bench "step" = one launch of the persistent
step-loop kernel advancing every scenario by `--emt-steps` (default 1000) EMT
passes, i.e. 50 ms of simulated time; the default K + W covers 1.15 s.

value  = total scenario-steps / max-over-ranks device time of the K timed
         launches (CUDA events on the engine's stream, L2 flushed between launches).
e2e    = the same metric through the C ABI with HOST buffers (batch H2D from
         pinned memory, S passes, waveform rows D2H), per step.
parity = every sample of the device run (warm-up + timed passes, all lanes)
         against the reference itself (oracle/_ref/libemtref.so, emtgrid::interpret
         on lane shards; the C oracle for C4), which also gives cpu_baseline.
The reference arm (--impl reference) runs the reference library over the same
lanes and pass window on all host cores, as BASELINE.md §2 prescribes.
"""
from __future__ import annotations

import argparse
import gzip
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DATA = os.path.join(ROOT, "paper_1903_01081_b200", "data")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def load_case(name="ieee39"):
    from paper_1903_01081_b200 import schedule as sch
    s = gzip.open(os.path.join(DATA, f"{name}.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(DATA, f"{name}.state.gz"), "rt").read())
    ids = json.load(open(os.path.join(DATA, f"{name}.json")))["component_ids"]
    return s, st, ids


def load_scale_case(k: int):
    """gen_scale_case(feeder33_pv3, k) as compiled by the reference (tools/make_scale_cases.py)."""
    from paper_1903_01081_b200 import schedule as sch
    s = gzip.open(os.path.join(DATA, f"feeder_scale{k}.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(DATA, f"feeder_scale{k}.state.gz"), "rt").read())
    return s, st


WORKLOADS = {
    "c3": ("ieee39-n1-sweep (BASELINE C3)", "ieee39", 1000),
    "c5": ("feeder33-pv-sweep shared G (BASELINE C5)", "feeder33_pv3", 4096),
    "c2": ("ieee39 single scenario (BASELINE C2)", "ieee39", 1),
    "c4": ("ieee39 x120 line-coupled single system, split at Bergeron lines (BASELINE C4)", "ieee39_c4", 120),
    # the reference's own large-scale case (gen_scale_case, proj/src/bench.cpp:54-117):
    # k feeder copies joined at the root node, one system, --scenarios = k (replicas only across GPUs)
    "scale": ("gen_scale_case(feeder33_pv3, k) single large system (reference format)", "feeder_scale", 128),
}


METRIC = {"c3": "scenario-steps/sec for N-1 EMT batch", "c5": "scenario-steps/sec for shared-G EMT batch",
          "c2": "us per time step on single case", "c4": "us per time step on large single case",
          "scale": "us per time step on large single case"}


def build_batch(scenarios: int, lo: int = 0, hi: int = -1, workload: str = "c3"):
    """Lanes [lo, hi) of a `scenarios`-lane sweep: C3 = N-1 breaker outages
    (sharding.n1_sweep), C5 = PV irradiance x temperature grid (shared G,
    gen_scenarios rows, proj/src/bench.cpp:119-149), C2 = the base case."""
    from paper_1903_01081_b200 import schedule as sch
    from paper_1903_01081_b200 import sharding
    hi = scenarios if hi < 0 else hi
    if workload == "c5":
        s, st, _ = load_case("feeder33_pv3")
        pvm = json.load(open(os.path.join(DATA, "feeder33_pv3.json")))["pv_sweep"]
        n = max(1, int(round(scenarios ** 0.5)))
        grid = sch.pv_grid(n, (scenarios + n - 1) // n)
        while len(grid) < scenarios:  # weak scaling beyond a square grid: shifted repeats
            grid += [(i + 1e-3 * len(grid), t) for i, t in grid[: scenarios - len(grid)]]
        return sch.pv_sweep_batch(s, st, pvm, grid[lo:hi]), sch.parse_info(s)
    if workload == "scale":  # one lane: gen_scale_case with k = scenarios, compiled by the reference
        s, st = load_scale_case(scenarios)
        return sch.Batch(s, sch.parse_info(s).const_table, st, 1), sch.parse_info(s)
    if workload == "c4":  # one system of `scenarios` IEEE-39 copies (one lane each) coupled by lines
        from paper_1903_01081_b200 import lines
        s, st, ids = load_case("ieee39_c4")
        return lines.c4_batch(s, st, ids, scenarios), sch.parse_info(s)
    s, st, ids = load_case("ieee39")
    if workload == "c2":
        return sch.n1_batch(s, st, ids, [("sw00", 1e9)] * (hi - lo)), sch.parse_info(s)
    scen = [(f"sw{b:02d}", tf) for b, tf in sharding.n1_sweep(scenarios)[lo:hi]]
    return sch.n1_batch(s, st, ids, scen), sch.parse_info(s)


def fp64_gemm_peak(dev) -> float:
    """Measured FP64 GEMM rate (TFLOP/s) of this GPU: torch.matmul (cuBLAS DGEMM), 8192^3, best of 10."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = a @ b
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b, c
    return 2.0 * n ** 3 / best / 1e12


def algorithmic_bytes_per_scenario_step(info, batch, shared_g: bool = False) -> float:
    """B = 8 [2 (n + m + S_blk + 2 N_sw + N_latch) + F_lane + C_var + K];
    F_lane = l_nnz + u_nnz for per-lane factors, else 0 plus the shared factor 8 (l+u) / W."""
    text = batch.schedule
    lines = text.splitlines()
    mat = next(l for l in lines if l.startswith("MATRIX")).split()
    lnnz = int(mat[3].split("=")[1])
    unnz = int(mat[4].split("=")[1])
    n_sw = sum(1 for p in info.procs if p.code == 7)
    s_blk = sum(p.state_len for p in info.procs if p.kind >= 4)
    n_latch = sum(1 for l in lines if l.startswith("LATCH"))
    ct = batch.const_table
    c_var = int(np.sum(np.any(ct != ct[:, :1], axis=1)))
    k = len(info.channels)
    f_lane = 0 if shared_g else lnnz + unnz
    shared = 8.0 * (lnnz + unnz) / batch.width if shared_g else 0.0
    return 8 * (2 * (info.nodes + info.comps + s_blk + 2 * n_sw + n_latch) + f_lane + c_var + k) + shared


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for ln in open(self.path):
                f = [x.strip() for x in ln.split(",")]
                if len(f) >= 9:
                    rows.append(f)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        load = [x for x in sm if x > 0.5 * (max(smax) if smax else 1)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def bench_config(args, W, per_gpu, world, info):
    """The workload description both arms print (`config`): identical for the device arm
    and the reference arm, so the two lines describe the same workload."""
    return {"workload": WORKLOADS[args.workload][0], "scenarios": W, "scenarios_per_gpu": per_gpu,
            "emt_steps_per_bench_step": args.emt_steps if args.impl == "ours" else
            (args.cpu_emt_steps_per_step or args.emt_steps),
            "dt": info.dt, "nodes": info.nodes, "components": info.comps, "case": WORKLOADS[args.workload][1],
            "parallelism": (f"{W} line-coupled copies split over {world} GPU(s)" if args.workload == "c4"
                            else f"one k={args.scenarios} system per GPU (replicas only: the shared root "
                                 "node couples every copy into one LU)" if args.workload == "scale"
                            else f"{W} scenario lanes in contiguous shards over {world} GPU(s), no per-step traffic"),
            "l2": "flushed (256 MiB write) between timed launches"}


def flush_l2(torch, buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1903_01081_b200 import engine

    rank, world, local = dist_env()
    if "DEVELOPER" in engine.lib().emt_version().decode() and not args.allow_dev_build:
        raise SystemExit("bench.py: libemtb200.so is a developer build (EMTB200_* knobs live); rebuild with "
                         "paper_1903_01081_b200/build.py --force or pass --allow-dev-build")
    if world > 1:
        # BENCH_DIST_BACKEND=gloo + BENCH_SHARE_GPU=1 lets the multi-rank control flow be
        # exercised with several ranks on one GPU (NCCL refuses duplicate devices)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if os.environ.get("BENCH_SHARE_GPU") == "1":
        local = 0
    cdev = None if world > 1 and dist.get_backend() == "gloo" else local  # collectives' tensor device
    torch.cuda.set_device(local)
    dev = local

    from paper_1903_01081_b200 import sharding
    wl_name, _, _ = WORKLOADS[args.workload]
    # strong scaling (default, BASELINE C3 "1000 scenarios sharded over 1/2/4/8"): the
    # `--scenarios` lanes are split into contiguous shards, one per GPU; weak scaling
    # (`--scaling weak`): `--scenarios` per GPU. C4 is ONE system of `--scenarios`
    # line-coupled copies split over the GPUs (always strong).
    weak = args.scaling == "weak" and args.workload not in ("c4", "scale")
    W = args.scenarios * world if weak else args.scenarios
    if args.workload == "scale":  # one unsplittable system (shared root node): replicas only, one per GPU
        batch, info = build_batch(args.scenarios, workload="scale")
        W, lo, hi = 1, 0, 1
    else:
        lo, hi = sharding.shard_bounds(W, world, rank)
        batch, info = build_batch(W, lo, hi, args.workload)
    S = args.emt_steps
    total_steps = (args.warmup + args.steps) * S

    kern = {"auto": engine.KERNEL_AUTO, "specialised": engine.KERNEL_SPECIALISED,
            "generic": engine.KERNEL_GENERIC}[args.kernel]
    if args.workload == "c4":  # lane shard + line-end ring exchange every K-1 passes
        runner = sharding.LineSplitShard(dist if world > 1 else None, batch, lo, hi, device=dev, kernel=kern,
                                         warps=args.warps)
        eng, adv = runner.eng, runner.advance
    else:
        eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width,
                            device=dev, kernel=kern, warps=args.warps, tensor_solve=args.tensor_solve)
        adv = eng.advance
    eng.reserve(total_steps)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    for _ in range(args.warmup):
        adv(S)
    eng.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = eng.stats().kernel_launches
    with ClockSampler(dev) as clocks:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush_l2(torch, flush)
                starts[k].record(stream)
            adv(S)
            ends[k].record(stream)
        eng.sync()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_launch_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    local_ms = sum(per_launch_ms)
    st = eng.stats()
    launches_timed = st.kernel_launches - launches0
    last = eng.waves(total_steps - S, S).values
    fc_local, steps_local = st.factor_count, eng.refactor_steps()
    # every pass of the run (warm-up + timed) for the parity check against the reference
    all_waves = eng.waves(0, total_steps).values if (world == 1 and not args.skip_cpu) else None

    # ---- e2e through the public API with HOST buffers, rank-local shard. The engine
    # (schedule parse + code generation + JIT, the analogue of compile_task, which the
    # reference's timed_run also leaves outside its clock, proj/src/bench.cpp:157-181) is
    # built once; every step then loads its batch from pinned host memory (H2D of the
    # whole arena + constant table), runs S passes and streams the waveform rows back
    # into pinned host memory chunk by chunk (D2H overlapped with the next chunk).
    e2e_local, e2e_digest_ok = float('nan'), None
    cold = None
    if not args.skip_e2e and args.workload == "c4" and world > 1:
        # line-split across ranks: reload the shard from pinned host, step with the
        # exchange, read the shard's waveform rows back
        e2e_steps = max(3, args.steps)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        ct_host, init_host = pin(batch.const_table), pin(batch.initial)
        e2e_s = []
        for k in range(e2e_steps + 1):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            runner.reload(init_host, ct_host)
            eng.reserve(S)
            adv(S)
            host_w = eng.waves(0, S).values
            t1 = time.perf_counter()
            if k > 0:
                e2e_s.append(t1 - t0)
        e2e_local = statistics.median(e2e_s)
        e2e_digest_ok = None
    elif not args.skip_e2e:
        e2e_steps = max(3, args.steps)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        ct_host = pin(batch.const_table)
        init_host = pin(batch.initial)
        # Two engines take turns: batch k computes on one while batch k-1's last waveform
        # chunk drains to the host from the other and batch k+1's H2D is staged; compute
        # stays serialised (each commit waits for the other engine's last launch).
        bufs = [torch.empty((S, len(info.channels) * (hi - lo)), dtype=torch.float64, pin_memory=True).numpy()
                for _ in range(2)]
        engs = [engine.Engine(batch.schedule, init_host, const_table=ct_host, width=batch.width, device=dev,
                              kernel=kern, warps=args.warps, tensor_solve=args.tensor_solve) for _ in range(2)]
        streams = [torch.cuda.ExternalStream(x.stream_ptr(), device=dev) for x in engs]
        for x in engs:
            x.reserve(S)

        def e2e_run(nsteps):
            done = [None, None]
            engs[0].stage(init_host, ct_host)
            for k in range(nsteps):
                E, O = k % 2, (k + 1) % 2
                if k >= 2:
                    engs[E].wait()
                if done[O] is not None:
                    streams[E].wait_event(done[O])
                engs[E].commit()
                if k + 1 < nsteps:
                    engs[O].stage(init_host, ct_host)
                engs[E].run_async(S, bufs[E], chunk=args.e2e_chunk)
                ev = torch.cuda.Event()
                ev.record(streams[E])
                done[E] = ev
            for x in engs:
                x.wait()
            return bufs[(nsteps - 1) % 2]

        e2e_run(2)  # warm-up: copy streams, events, staging buffers
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host_waves = e2e_run(e2e_steps)
        e2e_local = (time.perf_counter() - t0) / e2e_steps
        e2e_digest_ok = bool(np.array_equal(host_waves, eng.waves(0, S).values))
        for x in engs:
            x.close()
        if world == 1 and args.workload != "scale":
            # cold start: a fresh process with empty in-memory and on-disk cubin caches (JIT included)
            cold = {}
            for mode in ("sync", "async"):  # each in a fresh process with an empty cubin cache
                r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "cold_start.py"), args.workload,
                                    str(W), str(S), str(dev), mode], capture_output=True, text=True, timeout=600)
                try:
                    cold[mode] = json.loads(r.stdout.strip().splitlines()[-1])
                except (ValueError, IndexError):
                    cold = {"error": (r.stderr or r.stdout)[-300:]}
                    break

    if world > 1:
        max_ms = sharding.reduce_max(dist, local_ms, device=cdev)
        e2e_max = sharding.reduce_max(dist, e2e_local, device=cdev)
        # final result gather (the only inter-GPU traffic): per-rank digests + refactor steps
        digests = sharding.gather_digests(dist, sharding.digest(last), world, device=cdev)
        mx = int(sharding.reduce_max(dist, float(len(steps_local)), device=cdev))
        pad = np.full(max(mx, 1), -1.0)
        pad[: len(steps_local)] = steps_local
        tt = torch.tensor(pad, dtype=torch.float64, device=cdev)
        parts = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(parts, tt)
        fc = sharding.combine_factor_counts([[int(x) for x in p.cpu().numpy() if x >= 0] for p in parts])
    else:
        max_ms, e2e_max, fc = local_ms, e2e_local, fc_local
        digests = sharding.digest(last)[None, :]

    scen_steps = W * S * args.steps  # all ranks' lanes
    value = scen_steps / (max_ms * 1e-3)
    clk = clocks.summary()
    if rank == 0:
        peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
        peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
        bytes_per = algorithmic_bytes_per_scenario_step(info, batch, shared_g=args.workload == "c5")
        avg_launch_s = (local_ms / args.steps) * 1e-3
        lanes_local = hi - lo
        achieved = bytes_per * lanes_local * S / avg_launch_s / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):  # ncu --set full capture of the same kernel (tools/ncu_summary.py), per EMT step
            per_step = json.load(open(tp)).get("dram_bytes_per_emt_step")
            traffic = per_step * S * lanes_local / json.load(open(tp)).get("lanes", lanes_local) if per_step else None
        cpu, par = cpu_baseline(args, batch, all_waves, total_steps) if all_waves is not None else (None, None)
        del all_waves
        h2d = batch.const_table.nbytes + batch.initial.nbytes  # per bench step (S passes)
        d2h = S * len(info.channels) * (hi - lo) * 8
        metric, unit, hib, val, e2e_val = (METRIC[args.workload], "scenario-steps/s", True, value, W * S / e2e_max)
        if args.workload in ("c2", "c4", "scale"):  # latency of one system: µs per EMT time step
            metric, unit, hib = METRIC[args.workload], "us/step", False
            val, e2e_val = 1e3 * max_ms / (args.steps * S), 1e6 * e2e_max / S
        out = {
            "metric": metric,
            "value": val,
            "unit": unit,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": max_ms / args.steps,
            "higher_is_better": hib,
            "scaling": "weak" if weak else "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(args, W, hi - lo, world, info),
            "e2e": {"value": e2e_val, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "matches_device_run": e2e_digest_ok,
                    "note": "per step: the batch's H2D from pinned host (Engine.stage, overlapping the previous "
                            f"step's run) + Engine.commit + Engine.run_async (S passes, waveform rows D2H to pinned host in "
                            f"{args.e2e_chunk}-pass chunks overlapped with compute); two engines alternate so a batch's "
                            "last chunk drains while the next computes (compute serialised); engines built once "
                            "outside the clock; host wall time over all e2e steps / steps"},
            "gpu_launches": int(launches_timed),
            "kernel": eng.summary[:200],
            "factor_count": int(fc),
            "result_digest": digests.tolist(),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "bytes_per_scenario_step": bytes_per,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                         "note": "achieved = SURVEY §8(d) algorithmic bytes / launch time; the lane state stays in "
                                 "shared memory for a whole launch, so DRAM moves only `traffic` per launch and the "
                                 "kernel is bound by its per-pass instruction latency, not HBM (DESIGN.md §3.3)"},
            "clocks": clk,
        }
        if cold is not None and "sync" in cold:
            a_, s_ = cold["async"], cold["sync"]
            conv = (lambda sec: 1e6 * sec / S) if unit == "us/step" else (lambda sec: W * S / sec)
            out["e2e_cold"] = {"value": conv(a_["total_s"]), "unit": unit, "seconds": a_["total_s"],
                               "jit_s": a_["jit_s"], "kernel_during_step": a_["kernel_during_run"],
                               "sync_jit": {"value": conv(s_["total_s"]), "seconds": s_["total_s"],
                                            "jit_s": s_["jit_s"]},
                               "same_waves": a_["digest"] == s_["digest"],
                               "note": "one bench step from a fresh process with empty cubin caches, H2D + S passes + "
                                       "D2H included: `value` with EMT_FLAG_ASYNC_JIT (generic kernel while NVRTC "
                                       "compiles, then the specialised kernel), `sync_jit` with the compile first"}
        elif cold is not None:
            out["e2e_cold"] = cold
        if args.tensor_solve and "solve=dmma" in eng.summary:
            # the batched V = G^-1 I product on the FP64 tensor cores, 2 n^2 flops
            # per scenario-step, against this GPU's FP64 GEMM rate measured here (cuBLAS DGEMM
            # 8192^3, best of 10) since MEASURED_PEAKS.json holds no FP64 figure
            n = info.nodes
            dflops = 2.0 * n * n * lanes_local * S / avg_launch_s / 1e12
            dpeak = fp64_gemm_peak(cdev)
            out["roofline_dmma"] = {"bound": "tensor", "achieved": dflops, "peak": dpeak, "unit": "TFLOP/s",
                                    "frac": dflops / dpeak, "flops_per_scenario_step": 2.0 * n * n,
                                    "peak_source": "torch.matmul float64 8192^3 on this GPU, best of 10",
                                    "note": "the solve is one part of the pass: the kernel as a whole is in 'roofline'"}
        if args.workload == "scale":
            # the bound that matters: in the reference's order every backward row
            # subtracts its smallest column first, the row finished last, so with the shared root's
            # fill the sweep is ONE chain of u_nnz dependent FP64 subtractions; floor = u_nnz x the
            # dependent DADD latency (8.1 cycles, tools/micro/lat.cu on B200) at the sampled SM clock
            mat = next(l for l in batch.schedule.splitlines() if l.startswith("MATRIX")).split()
            unnz = int(mat[4].split("=")[1])
            mhz = clk.get("sm_mhz") or 1965.0
            floor_us = unnz * 8.1 / mhz
            out["roofline_chain"] = {"bound": "latency", "chain_ops": unnz, "dadd_latency_cycles": 8.1,
                                     "sm_mhz": mhz, "floor_us_per_step": floor_us, "achieved_us_per_step": val,
                                     "frac": floor_us / val,
                                     "note": "backward-sweep dependency chain of the reference's row order "
                                             "(sparse.cpp:161-170); HBM 'roofline' above is far from binding"}
        if cpu is not None:
            out["cpu_baseline"] = cpu
        if par is not None:
            out["parity"] = par
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------- reference (CPU) arm

def oracle_run(batch, steps: int, got=None):
    """C4 has no reference path (the reference has no line model): the C restatement
    (oracle/emt_oracle.c, the parity checker) on the whole coupled system, one thread —
    the copies are one system, so they cannot be sharded. Returns (seconds, parity)."""
    from oracle import oracle, parity
    sched = oracle.Schedule(batch.text())
    sched.interpret(batch.initial, 20)  # warm-up
    t0 = time.perf_counter()
    r = sched.interpret(batch.initial, steps)
    secs = time.perf_counter() - t0
    rep = parity.merge([parity.compare(got, r.waves)]) if got is not None else None
    return secs, rep


def cpu_baseline(args, batch, got, total_steps):
    """The reference on the box's host cores over the SAME lanes and passes the device
    just ran (warm-up + timed launches), timed over the timed passes, and every sample
    of the device run checked against it (oracle/parity.py). Returns (cpu_baseline, parity)."""
    from oracle import parity
    S = args.emt_steps
    W = batch.width
    if args.workload == "c4":
        secs, rep = oracle_run(batch, total_steps, got)
        rep.update({"against": "oracle/emt_oracle.c interpret (the reference has no line model)",
                    "lanes": W, "passes": total_steps})
        return ({"value": 1e6 * secs / total_steps, "unit": "us/step", "cores": 1, "kind": "port",
                 "sample": f"{W}-copy line-coupled system x {total_steps} EMT steps, oracle/emt_oracle.c "
                           "interpret (the reference has no line model), single thread"}, rep)
    res = parity.reference_sweep(batch, total_steps, got=got, warmup=S * args.warmup)
    rep = res["parity"]
    rep.update({"against": "reference emtgrid::interpret (oracle/_ref/libemtref.so) on lane shards",
                "lanes": W, "passes": total_steps})
    timed = S * args.steps
    if args.workload in ("c2", "scale"):
        cpu = {"value": 1e6 * res["seconds"] / timed, "unit": "us/step", "cores": 1, "kind": "reference",
               "sample": f"1 system x {total_steps} EMT steps ({S * args.warmup} warm-up), emtgrid::interpret "
                         "(oracle/_ref/libemtref.so), single thread"}
    else:
        cpu = {"value": W * timed / res["seconds"], "unit": "scenario-steps/s", "cores": res["procs"],
               "kind": "reference",
               "sample": f"{W} scenarios x {total_steps} EMT steps (the device run's passes; {S * args.warmup} "
                         f"warm-up outside the clock), emtgrid::interpret on {res['procs']} contiguous lane "
                         "shards, one process per core (oracle/_ref/libemtref.so)"}
    return cpu, rep


def run_reference(args):
    """The reference arm: the reference's own CPU implementation on the same workload,
    lanes and pass window as our arm (S passes per bench step, W warm-up + K timed steps)."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import parity
    S = args.cpu_emt_steps_per_step or args.emt_steps
    weak = args.scaling == "weak" and args.workload not in ("c4", "scale")
    W0 = args.scenarios * world if weak else args.scenarios
    batch, info = build_batch(W0, workload=args.workload)
    kind = "reference"
    if args.workload == "c4":
        kind, procs = "port", 1
        secs, _ = oracle_run(batch, S * args.steps)
        W = batch.width
    else:
        res = parity.reference_sweep(batch, S * (args.warmup + args.steps), warmup=S * args.warmup)
        W, secs, procs = batch.width, res["seconds"], res["procs"]
    metric, unit, hib, value = METRIC[args.workload], "scenario-steps/s", True, W * S * args.steps / secs
    if args.workload in ("c2", "c4", "scale"):
        metric, unit, hib, value = METRIC[args.workload], "us/step", False, 1e6 * secs / (S * args.steps)
    out = {
        "impl": "reference",
        "metric": metric,
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": hib,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args, W, W // world if args.workload not in ("scale",) else W, world, info),
        "cpu_baseline": {"value": value, "unit": unit, "cores": procs, "kind": kind,
                         "sample": f"{W} {'copies' if kind == 'port' else 'scenarios'} x {S} EMT steps per bench "
                                   f"step ({args.warmup} warm-up + {args.steps} timed, the passes our arm times), "
                                   + ("oracle/emt_oracle.c (no reference line model), one thread" if kind == "port"
                                      else "emtgrid::interpret (oracle/_ref/libemtref.so)")},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3",
                    help="c3 = IEEE-39 N-1 sweep (headline), c5 = feeder PV shared-G sweep, c2 = single scenario, "
                         "c4 = line-coupled 120-copy system, scale = gen_scale_case k (--scenarios) single system")
    ap.add_argument("--scenarios", type=int, default=None,
                    help="scenarios in total (strong scaling) or per GPU (--scaling weak)")
    ap.add_argument("--emt-steps", type=int, default=1000, help="EMT passes per bench step (one launch)")
    ap.add_argument("--cpu-emt-steps-per-step", type=int, default=0,
                    help="EMT passes per bench step in the reference arm (0 = --emt-steps, the same window)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: --scenarios lanes in total, sharded over the GPUs (BASELINE C3); "
                         "weak: --scenarios lanes per GPU")
    ap.add_argument("--e2e-chunk", type=int, default=1000, help="passes per launch in the e2e streaming run")
    ap.add_argument("--kernel", choices=["auto", "specialised", "generic"], default="auto")
    ap.add_argument("--warps", type=int, default=0, help="specialised kernel: warps per 32-lane group (0 = auto)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--tensor-solve", action="store_true",
                    help="shared-G batches (C5): V = G^-1 I on the FP64 tensor cores (amplitude-relative parity)")
    ap.add_argument("--skip-cpu", action="store_true", help="no cpu_baseline / parity leg")
    ap.add_argument("--allow-dev-build", action="store_true", help="run on a developer build (knobs live)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.scenarios is None:
        args.scenarios = WORKLOADS[args.workload][2]
    if args.workload == "scale" and args.emt_steps == 1000:
        args.emt_steps = 50  # k=128: ~8 ms per pass here and in the reference
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
