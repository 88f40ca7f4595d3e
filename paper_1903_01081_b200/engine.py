"""Python host API over libemtb200.so, mirroring the reference executor interface.

    interpret(schedule, initial, steps, options)          ~ emtgrid::interpret
        /root/reference/proj/include/emtgrid/exec.hpp:29-30, proj/src/exec.cpp:350-383
    execute_parallel(schedule, initial, workers, steps)   ~ emtgrid::execute_parallel
        proj/include/emtgrid/exec.hpp:36-37 (the device is the parallel executor)
    WaveformSet                                           ~ proj/include/emtgrid/waveform.hpp:12-37
    EmtError(code, where, message)                        ~ emtgrid::Error, proj/include/emtgrid/common.hpp:39-58

`schedule` is the reference's canonical `.cgmsched` text (ScheduleProgram::serialize)
and `initial` the flat extent*width arena (build_initial_arena / parse_state).
There is no CPU path: a missing or unloadable libemtb200.so raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import build as _build

ERROR_CODES = [
    "MalformedDocument", "UnknownComponentKind", "DanglingReference", "DuplicateIdentifier",
    "InvalidParameter", "ArityMismatch", "NonFiniteState", "SingularMatrix", "SingularSystem",
    "DimensionMismatch", "CycleDetected", "TopologyMismatch", "CapacityExceeded", "UnknownKind",
    "UnknownDialect", "ToolchainUnavailable", "CompilationFailed", "UnknownTask", "NotFinished",
    "NonPositiveInput", "IoError",
]


class EmtError(RuntimeError):
    """emtgrid::Error equivalent: ``code`` is the ErrorCode name, ``status`` the C status."""

    def __init__(self, status: int, detail: str):
        self.status = status
        if 1 <= status <= len(ERROR_CODES):
            self.code = ERROR_CODES[status - 1]
        elif status == 64:
            self.code = "CudaError"
        elif status == 66:
            self.code = "InexactDivision"
        else:
            self.code = f"Status{status}"
        self.detail = detail
        super().__init__(f"{self.code}: {detail}")


class _Config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("lane_begin", ctypes.c_int32), ("lane_count", ctypes.c_int32),
                ("lanes_per_block", ctypes.c_int32), ("warps_per_group", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32)]


KERNEL_AUTO, KERNEL_SPECIALISED, KERNEL_GENERIC, KERNEL_TSIMT, KERNEL_SYSTEM = 0, 1, 2, 3, 4
FLAG_TENSOR_SOLVE = 1
FLAG_EXACT_DIVISION = 2  # IEEE fallback in every backward row (include/emt_b200.h)
FLAG_ASYNC_JIT = 4  # run the generic kernel while the specialised one compiles (include/emt_b200.h)


class _Options(ctypes.Structure):
    _fields_ = [("divergence_limit", ctypes.c_double), ("warmup_steps", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("factor_count", ctypes.c_int32), ("measured_steps", ctypes.c_int32),
                ("measured_seconds", ctypes.c_double), ("kernel_launches", ctypes.c_int32),
                ("switch_events", ctypes.c_int32)]


class _Event(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int32), ("lane", ctypes.c_int32), ("process", ctypes.c_int32)]


_lib = None


def library_path() -> str:
    return _build.LIB


def lib():
    """Loads the in-tree CUDA library; raises if it is absent (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_build.LIB):
            raise RuntimeError(f"{_build.LIB} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(_build.LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        vp = ctypes.c_void_p
        L.emt_last_error.restype = ctypes.c_char_p
        L.emt_version.restype = ctypes.c_char_p
        L.emt_interpret.argtypes = [ctypes.c_char_p, dp, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.POINTER(_Options), ctypes.POINTER(_Config), dp, dp,
                                    ctypes.POINTER(_Stats)]
        L.emt_execute_parallel.argtypes = [ctypes.c_char_p, dp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.POINTER(_Options), ctypes.POINTER(_Config), dp, dp,
                                           ctypes.POINTER(_Stats)]
        L.emt_create.argtypes = [ctypes.c_char_p, dp, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.POINTER(vp)]
        L.emt_run.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, dp, ctypes.POINTER(_Stats)]
        L.emt_error_detail.argtypes = [vp]
        L.emt_error_detail.restype = ctypes.c_char_p
        L.emt_destroy.argtypes = [vp]
        L.emt_engine_create.argtypes = [ctypes.c_char_p, dp, ctypes.c_int32, dp, ctypes.c_int64,
                                        ctypes.POINTER(_Config), ctypes.POINTER(vp)]
        L.emt_engine_destroy.argtypes = [vp]
        L.emt_engine_destroy.restype = None
        L.emt_engine_shape.argtypes = [vp] + [ip] * 9
        L.emt_engine_reserve.argtypes = [vp, ctypes.c_int32]
        L.emt_engine_advance.argtypes = [vp, ctypes.c_int32, ctypes.c_int32]
        L.emt_engine_sync.argtypes = [vp]
        L.emt_engine_read_waves.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, dp, dp]
        L.emt_engine_read_state.argtypes = [vp, dp]
        L.emt_engine_read_events.argtypes = [vp, ctypes.POINTER(_Event), ctypes.c_int32, ip]
        L.emt_engine_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
        L.emt_engine_device_waves.argtypes = [vp]
        L.emt_engine_device_waves.restype = vp
        L.emt_engine_stream.argtypes = [vp]
        L.emt_engine_stream.restype = vp
        L.emt_engine_read_refactor_steps.argtypes = [vp, ip, ctypes.c_int32, ip]
        L.emt_engine_load.argtypes = [vp, dp, ctypes.c_int64, dp]
        L.emt_engine_stage.argtypes = [vp, dp, ctypes.c_int64, dp]
        L.emt_engine_commit.argtypes = [vp]
        L.emt_engine_run.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, dp]
        L.emt_engine_run_async.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, dp]
        L.emt_engine_wait.argtypes = [vp]
        L.emt_engine_profile.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]
        L.emt_engine_ring.argtypes = [vp, ctypes.POINTER(vp), ip, ip, ip]
        L.emt_engine_attach_ring.argtypes = [vp, vp]
        L.emt_engine_attach_lines.argtypes = [vp, vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.emt_ipc_alloc.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(vp), ctypes.c_char_p]
        L.emt_ipc_open.argtypes = [ctypes.c_int32, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.emt_ipc_close.argtypes = [vp]
        L.emt_ipc_free.argtypes = [vp]
        L.emt_engine_kernel.argtypes = [vp]
        L.emt_engine_kernel.restype = ctypes.c_int32
        L.emt_engine_wait_jit.argtypes = [vp]
        L.emt_engine_source.argtypes = [vp]
        L.emt_engine_source.restype = ctypes.c_char_p
        L.emt_engine_summary.argtypes = [vp]
        L.emt_engine_summary.restype = ctypes.c_char_p
        L.emt_codegen.argtypes = [ctypes.c_char_p, dp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_char_p)]
        L.emt_waves_to_text.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_int32, ctypes.c_int32, dp, dp,
                                        ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int64)]
        L.emt_source_cos.argtypes = [ctypes.c_int32, dp, dp, ctypes.c_int64]
        L.emt_engine_ctas.argtypes = [vp, ip, ip]
        L.emt_emit_program.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
        L.emt_free.argtypes = [vp]
        L.emt_free.restype = None
        _lib = L
    return _lib


EXPORTED_SYMBOLS = [
    "emt_interpret", "emt_last_error", "emt_engine_create", "emt_engine_destroy", "emt_engine_shape",
    "emt_engine_reserve", "emt_engine_advance", "emt_engine_sync", "emt_engine_read_waves",
    "emt_engine_read_state", "emt_engine_read_events", "emt_engine_stats", "emt_engine_device_waves",
    "emt_engine_stream", "emt_version", "emt_engine_kernel", "emt_engine_wait_jit", "emt_engine_source", "emt_engine_summary",
    "emt_codegen", "emt_engine_read_refactor_steps", "emt_engine_load", "emt_engine_run",
    "emt_engine_ring", "emt_engine_attach_ring", "emt_engine_stage", "emt_engine_commit",
    "emt_engine_profile", "emt_engine_run_async", "emt_engine_wait",
    "emt_engine_attach_lines", "emt_ipc_alloc", "emt_ipc_open", "emt_ipc_close", "emt_ipc_free",
    "emt_waves_to_text", "emt_free", "emt_source_cos", "emt_engine_ctas", "emt_emit_program",
]


def emit_program(schedule: str) -> str:
    """emit_source(schedule, "sm100a"): a standalone CUDA program (emt_emit_program)."""
    out = ctypes.c_void_p()
    _check(lib().emt_emit_program(schedule.encode(), ctypes.byref(out)))
    try:
        return ctypes.cast(out, ctypes.c_char_p).value.decode()
    finally:
        lib().emt_free(out)


def device_cos(x: np.ndarray, device: int = 0) -> np.ndarray:
    """cos as the engine evaluates AC sources on the device (emt_source_cos)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    _check(lib().emt_source_cos(device, _dp(x), _dp(y), x.size))
    return y


def _check(status: int) -> None:
    if status != 0:
        raise EmtError(status, lib().emt_last_error().decode(errors="replace"))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def channel_names(schedule: str) -> List[str]:
    return [ln.split()[1] for ln in schedule.splitlines() if ln.startswith("CHANNEL ")]


def schedule_dt(schedule: str) -> float:
    """dt of the META record (%.17g, so the parsed double is the reference's)."""
    for ln in schedule.splitlines():
        if ln.startswith("META "):
            return float(next(f for f in ln.split() if f.startswith("dt=")).split("=")[1])
    raise ValueError("schedule has no META record")


def schedule_width(schedule: str) -> int:
    head = schedule.split("\n", 1)[0].split()
    return int(next(t for t in head if t.startswith("width=")).split("=")[1])


@dataclass
class ExecStats:
    factor_count: int = 0
    measured_seconds: float = 0.0
    measured_steps: int = 0
    kernel_launches: int = 0
    switch_events: int = 0


@dataclass
class ExecOptions:
    divergence_limit: float = 1e12
    warmup_steps: int = 0
    stats: Optional[ExecStats] = None


@dataclass
class WaveformSet:
    """Recorded channels; values rows = steps, column = channel*width + lane."""
    channels: List[str]
    width: int
    time: np.ndarray
    values: np.ndarray

    def steps(self) -> int:
        return len(self.time)

    def at(self, step: int, channel: int, lane: int = 0) -> float:
        return float(self.values[step, channel * self.width + lane])

    def lane(self, lane: int) -> "WaveformSet":
        cols = [c * self.width + lane for c in range(len(self.channels))]
        return WaveformSet(list(self.channels), 1, self.time.copy(), self.values[:, cols].copy())

    def to_text(self, threads: int = 0) -> str:
        """WaveformSet::to_text (proj/src/waveform.cpp:22-42): %.17g rows, formatted
        natively by emt_waves_to_text on `threads` host threads (0: all cores)."""
        return waves_to_text(self.channels, self.width, self.time, self.values, threads).decode()


def waves_to_text(channels: List[str], width: int, time: np.ndarray, values: np.ndarray, threads: int = 0) -> bytes:
    """The reference's waveform text (WaveformSet::to_text) of host rows, as bytes."""
    L = lib()
    t = np.ascontiguousarray(time, dtype=np.float64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.size != t.size * len(channels) * width:
        raise ValueError("values must hold rows x channels x width doubles")
    names = (ctypes.c_char_p * max(1, len(channels)))(*[c.encode() for c in channels])
    out, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(L.emt_waves_to_text(names, len(channels), int(width), _dp(t), _dp(v), t.size,
                               int(threads) if threads > 0 else (os.cpu_count() or 1), ctypes.byref(out), ctypes.byref(n)))
    try:
        return ctypes.string_at(out.value, n.value)
    finally:
        L.emt_free(out)


def _config(device: int = 0, lane_begin: int = 0, lane_count: int = 0, lanes_per_block: int = 0,
            warps: int = 0, kernel: int = KERNEL_AUTO, flags: int = 0) -> _Config:
    c = _Config()
    c.device, c.lane_begin, c.lane_count, c.lanes_per_block = device, lane_begin, lane_count, lanes_per_block
    c.warps_per_group, c.kernel, c.flags = warps, kernel, flags
    return c


def ipc_alloc(device: int, nbytes: int):
    """(device pointer, 64-byte IPC handle) of a zeroed allocation shareable with other processes."""
    p = ctypes.c_void_p()
    h = ctypes.create_string_buffer(64)
    _check(lib().emt_ipc_alloc(int(device), int(nbytes), ctypes.byref(p), h))
    return int(p.value), bytes(h.raw)


def ipc_open(device: int, handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(lib().emt_ipc_open(int(device), handle, ctypes.byref(p)))
    return int(p.value)


def codegen(schedule: str, const_table: Optional[np.ndarray] = None, width: int = 0, warps: int = 4,
            compile: bool = False, arch: str = "sm_100a"):
    """Generated kernel source + plan summary for a schedule (no GPU needed)."""
    L = lib()
    ct = None if const_table is None else np.ascontiguousarray(const_table, dtype=np.float64)
    src, summ = ctypes.c_char_p(), ctypes.c_char_p()
    _check(L.emt_codegen(schedule.encode(), _dp(ct) if ct is not None else None, int(width), int(warps),
                         1 if compile else 0, arch.encode(), ctypes.byref(src), ctypes.byref(summ)))
    return src.value.decode(), summ.value.decode()


def run_devices(schedule: str, initial: np.ndarray, steps: int, devices: Sequence[int] = (0,), warmup: int = 0):
    """The multi-device executor (emt_create / emt_run): the batch's lanes in
    contiguous shards over `devices`, run concurrently; returns (WaveformSet, ExecStats)."""
    L = lib()
    init = np.ascontiguousarray(initial, dtype=np.float64)
    width = schedule_width(schedule)
    extent = init.size // width
    h = ctypes.c_void_p()
    devs = (ctypes.c_int32 * len(devices))(*devices)
    _check(L.emt_create(schedule.encode(), _dp(init), extent, width, devs, len(devices), ctypes.byref(h)))
    try:
        nch = len(channel_names(schedule))
        waves = np.zeros((steps, nch * width))
        st = _Stats()
        rc = L.emt_run(h, steps, warmup, _dp(waves), ctypes.byref(st))
        if rc != 0:
            raise EmtError(rc, L.emt_error_detail(h).decode(errors="replace"))
    finally:
        L.emt_destroy(h)
    dt = schedule_dt(schedule)
    time = (np.arange(steps, dtype=np.float64) + 1.0) * dt
    return (WaveformSet(channel_names(schedule), width, time, waves),
            ExecStats(st.factor_count, st.measured_seconds, st.measured_steps, st.kernel_launches, st.switch_events))


def interpret(schedule: str, initial: np.ndarray, steps: int, options: Optional[ExecOptions] = None,
              device: int = 0, kernel: int = KERNEL_AUTO, warps: int = 0) -> WaveformSet:
    """Drop-in for emtgrid::interpret on the B200 (one-shot: upload, run, download)."""
    L = lib()
    init = np.ascontiguousarray(initial, dtype=np.float64)
    width = schedule_width(schedule)
    names = channel_names(schedule)
    waves = np.zeros((max(steps, 0), len(names) * width))
    time = np.zeros(max(steps, 0))
    opt = _Options()
    opt.divergence_limit = options.divergence_limit if options else 1e12
    opt.warmup_steps = options.warmup_steps if options else 0
    st = _Stats()
    cfg = _config(device, warps=warps, kernel=kernel)
    _check(L.emt_interpret(schedule.encode(), _dp(init), init.size, steps, ctypes.byref(opt), ctypes.byref(cfg),
                           _dp(waves), _dp(time), ctypes.byref(st)))
    if options is not None and options.stats is not None:
        s = options.stats
        s.factor_count, s.measured_seconds, s.measured_steps = st.factor_count, st.measured_seconds, st.measured_steps
        s.kernel_launches, s.switch_events = st.kernel_launches, st.switch_events
    return WaveformSet(names, width, time, waves)


def execute_parallel(schedule: str, initial: np.ndarray, workers: int, steps: int,
                     options: Optional[ExecOptions] = None, device: int = 0) -> WaveformSet:
    """emtgrid::execute_parallel signature; the GPU is the parallel executor, so
    `workers` only keeps the reference's NonPositiveInput contract (exec.cpp:387-389)."""
    if workers < 1:
        raise EmtError(20, "worker count must be at least 1")
    return interpret(schedule, initial, steps, options, device)


class Engine:
    """Device-resident batch: create once, advance in chunks, read waveforms/state."""

    def __init__(self, schedule: str, initial: np.ndarray, const_table: Optional[np.ndarray] = None,
                 width: int = 0, device: int = 0, lane_begin: int = 0, lane_count: int = 0,
                 lanes_per_block: int = 0, warps: int = 0, kernel: int = KERNEL_AUTO, tensor_solve: bool = False,
                 exact_division: bool = False, async_jit: bool = False):
        L = lib()
        self._h = ctypes.c_void_p()
        init = np.ascontiguousarray(initial, dtype=np.float64)
        ct = None if const_table is None else np.ascontiguousarray(const_table, dtype=np.float64)
        cfg = _config(device, lane_begin, lane_count, lanes_per_block, warps, kernel,
                      (FLAG_TENSOR_SOLVE if tensor_solve else 0) | (FLAG_EXACT_DIVISION if exact_division else 0)
                      | (FLAG_ASYNC_JIT if async_jit else 0))
        _check(L.emt_engine_create(schedule.encode(), _dp(ct) if ct is not None else None, int(width), _dp(init),
                                   init.size, ctypes.byref(cfg), ctypes.byref(self._h)))
        vals = [ctypes.c_int32() for _ in range(9)]
        _check(L.emt_engine_shape(self._h, *[ctypes.byref(v) for v in vals]))
        (self.lanes, self.channels, self.extent, self.consts, self.default_steps, self.nodes, self.l_nnz,
         self.u_nnz, self.layers) = (v.value for v in vals)
        self.channel_names = channel_names(schedule)
        self.rows = 0

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            lib().emt_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reserve(self, capacity_steps: int) -> None:
        _check(lib().emt_engine_reserve(self._h, int(capacity_steps)))
        self.rows = 0

    def advance(self, steps: int, sync: bool = False) -> None:
        _check(lib().emt_engine_advance(self._h, int(steps), 1 if sync else 0))
        self.rows += steps

    def load(self, initial: np.ndarray, const_table: Optional[np.ndarray] = None) -> None:
        """New batch from host buffers (whole-batch arena / const table); rewinds to pass 0.
        Pass pinned arrays (e.g. torch pin_memory().numpy()) for asynchronous H2D."""
        init = np.ascontiguousarray(initial, dtype=np.float64)
        ct = None if const_table is None else np.ascontiguousarray(const_table, dtype=np.float64)
        _check(lib().emt_engine_load(self._h, _dp(init), init.size, _dp(ct) if ct is not None else None))
        self.rows = 0

    def stage(self, initial: np.ndarray, const_table: Optional[np.ndarray] = None) -> None:
        """Start uploading the next batch (pinned host arrays: asynchronous); see commit()."""
        init = np.ascontiguousarray(initial, dtype=np.float64)
        ct = None if const_table is None else np.ascontiguousarray(const_table, dtype=np.float64)
        self._staged = (init, ct)  # keep the host buffers alive until the copy ran
        _check(lib().emt_engine_stage(self._h, _dp(init), init.size, _dp(ct) if ct is not None else None))

    def commit(self) -> None:
        """Make the staged batch current (device copy, stream-ordered) and rewind to pass 0."""
        _check(lib().emt_engine_commit(self._h))
        self.rows = 0

    def run(self, steps: int, out: Optional[np.ndarray] = None, chunk: int = 0) -> Optional[np.ndarray]:
        """Advance `steps` passes, streaming waveform rows into `out` (steps x channels*lanes,
        C-contiguous float64; pinned for overlap) chunk by chunk while the next chunk computes."""
        if out is not None:
            assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= steps * self.channels * self.lanes
        _check(lib().emt_engine_run(self._h, int(steps), int(chunk), _dp(out) if out is not None else None))
        self.rows += steps
        return out

    def profile(self) -> np.ndarray:
        """(32 warps x 64 markers) cycle sums of the phase profiler (EMTB200_CG_PROF=1 builds)."""
        buf = np.zeros(32 * 64, dtype=np.int64)
        _check(lib().emt_engine_profile(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), buf.size))
        return buf.reshape(32, 64)

    def ring(self):
        """(device pointer, lanes, cols, max passes per launch) of the line-end history mirror."""
        p = ctypes.c_void_p()
        lanes, cols, mc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().emt_engine_ring(self._h, ctypes.byref(p), ctypes.byref(lanes), ctypes.byref(cols), ctypes.byref(mc)))
        return int(p.value or 0), lanes.value, cols.value, mc.value

    def attach_ring(self, device_ptr: int) -> None:
        _check(lib().emt_engine_attach_ring(self._h, ctypes.c_void_p(device_ptr)))

    def run_async(self, steps: int, out: np.ndarray, chunk: int = 0) -> None:
        """run() without the final wait (call wait() before touching `out` or reloading)."""
        assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= steps * self.channels * self.lanes
        self._async_out = out
        _check(lib().emt_engine_run_async(self._h, int(steps), int(chunk), _dp(out)))
        self.rows += steps

    def wait(self) -> None:
        _check(lib().emt_engine_wait(self._h))
        self._async_out = None

    def attach_lines(self, mirror_ptr: int, progress_ptr: int, cta_offset: int, total_ctas: int,
                     system_scope: bool = False) -> None:
        """Device-side line exchange with other engines sharing `mirror` / `progress` (emt_engine_attach_lines)."""
        _check(lib().emt_engine_attach_lines(self._h, ctypes.c_void_p(mirror_ptr), ctypes.c_void_p(progress_ptr),
                                             int(cta_offset), int(total_ctas), 1 if system_scope else 0))

    def ctas(self):
        """(CTAs of this engine's launches, lanes per CTA; 0 for the generic kernel) — emt_engine_ctas."""
        c, l = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().emt_engine_ctas(self._h, ctypes.byref(c), ctypes.byref(l)))
        return c.value, l.value

    def sync(self) -> None:
        _check(lib().emt_engine_sync(self._h))

    def waves(self, row0: int = 0, rows: Optional[int] = None) -> WaveformSet:
        rows = self.rows - row0 if rows is None else rows
        v = np.zeros((rows, self.channels * self.lanes))
        t = np.zeros(rows)
        _check(lib().emt_engine_read_waves(self._h, row0, rows, _dp(v), _dp(t)))
        return WaveformSet(list(self.channel_names), self.lanes, t, v)

    def state(self) -> np.ndarray:
        a = np.zeros(self.extent * self.lanes)
        _check(lib().emt_engine_read_state(self._h, _dp(a)))
        return a

    def events(self, max_events: int = 1 << 16) -> np.ndarray:
        buf = (_Event * max_events)()
        n = ctypes.c_int32()
        _check(lib().emt_engine_read_events(self._h, buf, max_events, ctypes.byref(n)))
        k = min(n.value, max_events)
        return np.array([(buf[i].step, buf[i].lane, buf[i].process) for i in range(k)], dtype=np.int32).reshape(-1, 3)

    def refactor_steps(self, max_steps: int = 1 << 20) -> np.ndarray:
        buf = np.zeros(max_steps, dtype=np.int32)
        n = ctypes.c_int32()
        _check(lib().emt_engine_read_refactor_steps(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                                     max_steps, ctypes.byref(n)))
        return buf[: min(n.value, max_steps)].copy()

    def stats(self) -> ExecStats:
        st = _Stats()
        _check(lib().emt_engine_stats(self._h, ctypes.byref(st)))
        return ExecStats(st.factor_count, st.measured_seconds, st.measured_steps, st.kernel_launches,
                         st.switch_events)

    @property
    def kernel(self) -> int:
        return int(lib().emt_engine_kernel(self._h))

    def wait_jit(self) -> None:
        """Blocks until an asynchronous JIT (async_jit=True) is done; later launches use its kernel."""
        _check(lib().emt_engine_wait_jit(self._h))

    @property
    def summary(self) -> str:
        return lib().emt_engine_summary(self._h).decode()

    @property
    def source(self) -> str:
        return lib().emt_engine_source(self._h).decode()

    def device_waves_ptr(self) -> int:
        return int(lib().emt_engine_device_waves(self._h) or 0)

    def stream_ptr(self) -> int:
        return int(lib().emt_engine_stream(self._h) or 0)
