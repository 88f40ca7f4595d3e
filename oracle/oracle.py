"""ctypes bridge to oracle/libemtoracle.so — the plain-C restatement of the
reference's schedule executor (oracle/emt_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the CHECKER. The product package never
imports anything under oracle/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libemtoracle.so")
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, index: int = -1, lane: int = -1, step: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code  # 1 + emtgrid::ErrorCode
        self.msg = msg
        self.index, self.lane, self.step = index, lane, step


def build() -> None:
    subprocess.check_call(["make", "-s", "-C", _HERE, "oracle"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        L.emto_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p, ctypes.c_int]
        L.emto_free.argtypes = [ctypes.c_void_p]
        L.emto_shape.argtypes = [ctypes.c_void_p] + [ip] * 7
        L.emto_interpret.argtypes = [ctypes.c_void_p, dp, ctypes.c_int64, ctypes.c_int, dp, dp, ip, dp,
                                     ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ip, ip, ip, ip,
                                     ctypes.c_char_p, ctypes.c_int]
        _lib = L
    return _lib


@dataclass
class OracleRun:
    waves: np.ndarray          # steps x (channels*width)
    time: np.ndarray
    factor_count: int
    final_arena: np.ndarray
    events: np.ndarray         # (k, 3) int32: step, lane, process id


class Schedule:
    """A parsed schedule (ScheduleProgram::parse, proj/src/schedule.cpp:413)."""

    def __init__(self, text: str):
        L = lib()
        err = ctypes.create_string_buffer(4096)
        h = ctypes.c_void_p()
        rc = L.emto_parse(text.encode(), ctypes.byref(h), err, len(err))
        if rc != 0:
            raise OracleError(rc, err.value.decode())
        self._h = h
        vals = [ctypes.c_int() for _ in range(7)]
        L.emto_shape(h, *[ctypes.byref(v) for v in vals])
        (self.width, self.channels, self.extent, self.steps, self.nodes, self.l_nnz,
         self.u_nnz) = (v.value for v in vals)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().emto_free(self._h)
            self._h = None

    def interpret(self, initial: np.ndarray, steps: int, max_events: int = 1 << 16) -> OracleRun:
        """interpret (proj/src/exec.cpp:350-383)."""
        L = lib()
        init = np.ascontiguousarray(initial, dtype=np.float64)
        waves = np.zeros((steps, self.channels * self.width))
        time = np.zeros(steps)
        final = np.zeros(init.size)
        ev = np.zeros((max_events, 3), dtype=np.int32)
        fc, nev, ei, el, es = (ctypes.c_int() for _ in range(5))
        err = ctypes.create_string_buffer(4096)
        dp = ctypes.POINTER(ctypes.c_double)
        rc = L.emto_interpret(self._h, init.ctypes.data_as(dp), init.size, steps, waves.ctypes.data_as(dp),
                              time.ctypes.data_as(dp), ctypes.byref(fc), final.ctypes.data_as(dp),
                              ev.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), max_events, ctypes.byref(nev),
                              ctypes.byref(ei), ctypes.byref(el), ctypes.byref(es), err, len(err))
        if rc != 0:
            raise OracleError(rc, err.value.decode(), ei.value, el.value, es.value)
        return OracleRun(waves, time, fc.value, final, ev[: min(nev.value, max_events)].copy())
