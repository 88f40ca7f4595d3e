"""ctypes bridge to oracle/_ref/libemtref.so — the UNMODIFIED reference library.

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and the
CPU-baseline / reference arm of bench.py, never by the product package.
See oracle/ref_capi.cpp for which reference function each entry forwards to.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libemtref.so")
_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code  # 1 + emtgrid::ErrorCode
        self.msg = msg


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing (run `make -C oracle ref` where /root/reference exists)")
        L = ctypes.CDLL(LIB_PATH)
        c_char_pp = ctypes.POINTER(ctypes.c_char_p)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        L.emtref_free.argtypes = [ctypes.c_void_p]
        L.emtref_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                     ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                     ip, ctypes.c_char_p, ctypes.c_int]
        L.emtref_schedule_shape.argtypes = [ctypes.c_char_p, ip, ip, ip, ip, ctypes.c_char_p, ctypes.c_int]
        L.emtref_execute.argtypes = [ctypes.c_char_p, dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, dp, dp, ip, dp, ctypes.c_char_p, ctypes.c_int]
        L.emtref_parse_state.argtypes = [ctypes.c_char_p, ctypes.POINTER(dp), ctypes.POINTER(ctypes.c_int64),
                                         ip, ctypes.c_char_p, ctypes.c_int]
        L.emtref_run_serial.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, dp, dp, ip, ip, dp,
                                        ctypes.c_char_p, ctypes.c_int]
        L.emtref_document_shape.argtypes = [ctypes.c_char_p, ip, ip, ctypes.c_char_p, ctypes.c_int]
        L.emtref_gen_scale_case.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.c_char_p, ctypes.c_int]
        L.emtref_apply_overrides.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.c_char_p, ctypes.c_int]
        _lib = L
    return _lib


def _check(rc: int, err) -> None:
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"))


def _take_str(p: ctypes.c_void_p) -> str:
    s = ctypes.cast(p, ctypes.c_char_p).value.decode()
    lib().emtref_free(p)
    return s


@dataclass
class Compiled:
    schedule: str
    state: str
    loop_insertions: int


def compile_document(document: str, rows=None, profile: str = "cpu-serial") -> Compiled:
    """parse_model -> compile_task (proj/src/pipeline.cpp:5-18)."""
    L = lib()
    err = ctypes.create_string_buffer(4096)
    sp, st = ctypes.c_void_p(), ctypes.c_void_p()
    ins = ctypes.c_int(0)
    rows_json = json.dumps(rows).encode() if rows is not None else None
    rc = L.emtref_compile(document.encode(), profile.encode(), rows_json, ctypes.byref(sp),
                          ctypes.byref(st), ctypes.byref(ins), err, len(err))
    _check(rc, err)
    return Compiled(_take_str(sp), _take_str(st), ins.value)


def parse_state(text: str) -> np.ndarray:
    L = lib()
    err = ctypes.create_string_buffer(4096)
    p = ctypes.POINTER(ctypes.c_double)()
    n = ctypes.c_int64(0)
    w = ctypes.c_int(0)
    _check(L.emtref_parse_state(text.encode(), ctypes.byref(p), ctypes.byref(n), ctypes.byref(w), err, len(err)), err)
    out = np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else np.zeros(0)
    L.emtref_free(ctypes.cast(p, ctypes.c_void_p))
    return out


def schedule_shape(schedule: str):
    L = lib()
    err = ctypes.create_string_buffer(4096)
    w, c, e, s = (ctypes.c_int() for _ in range(4))
    _check(L.emtref_schedule_shape(schedule.encode(), ctypes.byref(w), ctypes.byref(c), ctypes.byref(e),
                                   ctypes.byref(s), err, len(err)), err)
    return w.value, c.value, e.value, s.value


@dataclass
class RefRun:
    waves: np.ndarray   # steps x (channels*width), column = channel*width + lane
    time: np.ndarray
    factor_count: int
    measured_seconds: float


def execute(schedule: str, initial: np.ndarray, steps: int, warmup: int = 0, workers: int = 0) -> RefRun:
    """interpret (workers=0, proj/src/exec.cpp:350) or execute_parallel (proj/src/exec.cpp:385)."""
    L = lib()
    width, nch, extent, _ = schedule_shape(schedule)
    init = np.ascontiguousarray(initial, dtype=np.float64)
    waves = np.zeros((steps, nch * width))
    time = np.zeros(steps)
    fc = ctypes.c_int(0)
    secs = ctypes.c_double(0)
    err = ctypes.create_string_buffer(4096)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = L.emtref_execute(schedule.encode(), init.ctypes.data_as(dp), init.size, steps, warmup, workers,
                          waves.ctypes.data_as(dp), time.ctypes.data_as(dp), ctypes.byref(fc),
                          ctypes.byref(secs), err, len(err))
    _check(rc, err)
    return RefRun(waves, time, fc.value, secs.value)


def run_serial(document: str, steps: int, warmup: int = 0) -> RefRun:
    """run_serial (proj/src/kernels.cpp:687-902)."""
    L = lib()
    err = ctypes.create_string_buffer(4096)
    nch, dsteps = ctypes.c_int(), ctypes.c_int()
    _check(L.emtref_document_shape(document.encode(), ctypes.byref(nch), ctypes.byref(dsteps), err, len(err)), err)
    waves = np.zeros((steps, nch.value))
    time = np.zeros(steps)
    fc = ctypes.c_int(0)
    secs = ctypes.c_double(0)
    ch = ctypes.c_int(0)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = L.emtref_run_serial(document.encode(), steps, warmup, waves.ctypes.data_as(dp), time.ctypes.data_as(dp),
                             ctypes.byref(ch), ctypes.byref(fc), ctypes.byref(secs), err, len(err))
    _check(rc, err)
    return RefRun(waves, time, fc.value, secs.value)


def gen_scale_case(document: str, k: int) -> str:
    L = lib()
    err = ctypes.create_string_buffer(4096)
    out = ctypes.c_void_p()
    _check(L.emtref_gen_scale_case(document.encode(), k, ctypes.byref(out), err, len(err)), err)
    return _take_str(out)


def apply_overrides(document: str, row) -> str:
    L = lib()
    err = ctypes.create_string_buffer(4096)
    out = ctypes.c_void_p()
    _check(L.emtref_apply_overrides(document.encode(), json.dumps(row).encode(), ctypes.byref(out), err,
                                    len(err)), err)
    return _take_str(out)


def waves_text(channels, width: int, time: np.ndarray, values: np.ndarray) -> str:
    """WaveformSet::to_text (proj/src/waveform.cpp:22-42) of host rows."""
    L = lib()
    L.emtref_waves_text.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p, ctypes.c_int]
    t = np.ascontiguousarray(time, dtype=np.float64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    names = (ctypes.c_char_p * max(1, len(channels)))(*[c.encode() for c in channels])
    err = ctypes.create_string_buffer(4096)
    out = ctypes.c_void_p()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(L.emtref_waves_text(names, len(channels), int(width), t.ctypes.data_as(dp), v.ctypes.data_as(dp),
                               int(t.size), ctypes.byref(out), err, len(err)), err)
    return _take_str(out)
