"""Parity of device waveforms against the reference at benchmark scale.

TEST INFRASTRUCTURE ONLY: used by tests/ and by bench.py's cpu_baseline leg as
the CHECKER of a finished device run; the product package never imports it.

The reference (`oracle/_ref/libemtref.so`, the unmodified emtgrid library) runs
`interpret` (/root/reference/proj/src/exec.cpp:350-383) on contiguous lane
shards, one forked process per host core. Lanes of a batch
are independent, so a shard's waveform columns are exactly the full batch's
columns for those lanes (pinned by tests/test_schedule_host.py). Each worker
compares its shard with the device waveforms it inherited through fork, so no
waveform crosses a pipe.

Bar (north_star): |got - want| <= 1e-12 + 1e-9 |want| on every sample; the
report also counts bit-identical samples (the engine is designed to be
bit-identical, including cos: paper_1903_01081_b200/csrc/libmcos.cuh).
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

REL, ABS = 1e-9, 1e-12

_GOT = None  # device waveforms (rows x channels*width), inherited by the forked workers


def compare(got: np.ndarray, want: np.ndarray) -> dict:
    """Per-sample bar and bitwise equality of two equally shaped waveform blocks."""
    got = np.ascontiguousarray(got, dtype=np.float64)
    want = np.ascontiguousarray(want, dtype=np.float64)
    if got.shape != want.shape:
        return {"samples": int(want.size), "bitwise": 0, "fail": int(want.size), "max_abs_diff": float("inf"),
                "max_excess": float("inf"), "shape_mismatch": [list(got.shape), list(want.shape)]}
    bit = got.view(np.uint64) == want.view(np.uint64)
    d = np.abs(got - want)
    excess = d - (ABS + REL * np.abs(want))
    excess[bit] = -np.inf  # NaN == NaN bitwise counts as equal
    bad = ~(excess <= 0) & ~bit
    out = {"samples": int(want.size), "bitwise": int(bit.sum()), "fail": int(bad.sum()),
           "max_abs_diff": float(np.nanmax(np.where(bit, 0.0, d))) if want.size else 0.0,
           "max_excess": float(excess.max()) if want.size else float("-inf")}
    if not bit.all():  # first non-identical sample: (row, column) of this block
        r, c = np.argwhere(~bit)[0]
        out["first_diff"] = [int(r), int(c)]
    return out


def merge(parts) -> dict:
    out = {"samples": 0, "bitwise": 0, "fail": 0, "max_abs_diff": 0.0, "max_excess": float("-inf")}
    for p in parts:
        if "first_diff" in p and ("first_diff" not in out or p["first_diff"][0] < out["first_diff"][0]):
            out["first_diff"] = p["first_diff"]
        for k in ("samples", "bitwise", "fail"):
            out[k] += p[k]
        out["max_abs_diff"] = max(out["max_abs_diff"], p["max_abs_diff"])
        out["max_excess"] = max(out["max_excess"], p["max_excess"])
    out["bitwise_fraction"] = out["bitwise"] / out["samples"] if out["samples"] else 1.0
    out["ok"] = out["fail"] == 0
    return out


def shard(batch, lo, hi=None):
    """Schedule text + initial arena of lanes [lo, hi) (or of the lane index list `lo`)
    of a batch: same slots and constants, fewer lanes."""
    from paper_1903_01081_b200 import schedule as sch
    idx = slice(lo, hi) if hi is not None else np.asarray(lo)
    ct = np.ascontiguousarray(batch.const_table[:, idx])
    ext = batch.initial.size // batch.width
    init = batch.initial.reshape(ext, batch.width)[:, idx].reshape(-1)
    return sch.widen_text(batch.schedule, ct), np.ascontiguousarray(init)


def columns(lanes, width: int, nch: int) -> np.ndarray:
    """Waveform columns (channel-major, then lane) of the given lanes."""
    lanes = np.asarray(lanes)
    return np.concatenate([c * width + lanes for c in range(nch)])


def _worker(job):
    text, init, steps, warmup, lo, hi, width, nch = job
    from oracle import ref
    t0 = time.perf_counter()
    r = ref.execute(text, init, steps, warmup=warmup)
    wall = time.perf_counter() - t0
    rep = None
    if _GOT is not None:
        cols = columns(np.arange(lo, hi), width, nch)
        rows = min(steps, _GOT.shape[0])
        rep = compare(_GOT[:rows][:, cols], r.waves[:rows])
        rep["lanes"] = [lo, hi]
    return {"seconds": r.measured_seconds, "wall": wall, "factor_count": r.factor_count, "parity": rep,
            "time": r.time if lo == 0 else None}


def reference_sweep(batch, steps: int, procs: int = 0, got: np.ndarray | None = None, warmup: int = 0) -> dict:
    """Run the reference over every lane of `batch` for `steps` passes (the first `warmup`
    of them outside its clock), sharded over `procs` forked processes (0 = all cores), and
    compare with `got` (device waveforms of the same passes, rows x channels*width)."""
    global _GOT
    from oracle import ref
    ref.lib()  # load libemtref.so in this process before forking (visible to the driver)
    W = batch.width
    _, nch, _, _ = ref.schedule_shape(batch.schedule)
    procs = max(1, min(procs or os.cpu_count() or 1, W))
    bounds = [(p * W // procs, (p + 1) * W // procs) for p in range(procs)]
    jobs = []
    for lo, hi in bounds:
        text, init = shard(batch, lo, hi)
        jobs.append((text, init, steps, warmup, lo, hi, W, nch))
    _GOT = got
    try:
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            res = pool.map(_worker, jobs)
    finally:
        _GOT = None
    out = {"lanes": W, "steps": steps, "procs": procs, "seconds": max(r["seconds"] for r in res),
           "wall": max(r["wall"] for r in res), "factor_counts": [r["factor_count"] for r in res],
           "time": res[0]["time"]}
    if got is not None:
        out["parity"] = merge([r["parity"] for r in res])
    return out
