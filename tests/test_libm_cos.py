"""The device cos (csrc/libmcos.cuh) is glibc's cos operation for operation.

CPU part: the same source compiled for the host (tests/libm_cos_host.cpp, g++
-ffp-contract=off) equals the live libm bit for bit on every branch of the
algorithm, including every source argument of the benchmarked workloads, and
the correctly rounded value is NOT what libm returns (why CUDA's cos or a
correctly rounded cos would not give parity). GPU part: the device build equals
the host libm on the same arguments (tests/test_gpu_parity.py covers it through
whole waveforms as well).
"""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def host_lib():
    global _lib
    if _lib is None:
        out = os.path.join(tempfile.mkdtemp(prefix="libmcos"), "libmcos_host.so")
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", out,
                               os.path.join(HERE, "libm_cos_host.cpp")])
        _lib = ctypes.CDLL(out)
    return _lib


def _run(fn, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    fn(x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(x.size))
    return y


def arguments(n=1_000_000, seed=7):
    rng = np.random.default_rng(seed)
    dt, w = 5e-5, 2 * np.pi * 60
    t = np.arange(1, 1_200_001) * dt  # 60 s of passes
    parts = [
        rng.uniform(-2e-8, 2e-8, n // 10),                 # |x| < 2^-27 and just above
        rng.uniform(-0.86, 0.86, n),                       # table + Taylor cos
        rng.uniform(-2.43, 2.43, n),                       # pi/2 - |x| branch (incl. |a| < 0.126)
        rng.uniform(-1e4, 1e4, n),                         # reduced by pi/2
        rng.uniform(-1.05e8, 1.05e8, n // 2),              # up to the reduction limit
        np.exp(rng.uniform(-30, 18.4, n)) * rng.choice([-1.0, 1.0], n),
        np.repeat(np.arange(1, 200000) * (np.pi / 2), 3) + np.tile([-1e-16, 0.0, 1e-16], 199999),
        w * t + 0.3, w * t - 2.1,                          # 60 Hz sources as the engine forms w*t + p
    ]
    return np.concatenate(parts)


def test_replica_equals_libm_bitwise():
    L = host_lib()
    x = arguments()
    a, b = _run(L.replica_cos, x), _run(L.libm_cos, x)
    same = a.view(np.uint64) == b.view(np.uint64)
    assert same.all(), (int((~same).sum()), x[~same][:5])


def test_special_values():
    L = host_lib()
    x = np.array([0.0, -0.0, 5e-324, -1e-300, np.inf, -np.inf, np.nan, 1e300, 1.1e8])
    a, b = _run(L.replica_cos, x), _run(L.libm_cos, x)
    assert ((a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))).all()


def test_libm_is_not_correctly_rounded_on_these_arguments():
    """The reason the replica exists: a correctly rounded cos would differ from glibc."""
    mp = pytest.importorskip("mpmath")
    mp.mp.prec = 200
    L = host_lib()
    x = np.random.default_rng(3).uniform(-1e4, 1e4, 20000)
    b = _run(L.libm_cos, x)
    diff = sum(1 for xi, bi in zip(x, b) if float(mp.cos(mp.mpf(float(xi)))) != bi)
    assert diff > 0


@pytest.mark.gpu
def test_device_replica_equals_host_libm():
    """emt_src_kernel-style evaluation on the device vs the host libm, all branches."""
    import torch
    from paper_1903_01081_b200 import engine
    x = arguments(n=200_000, seed=11)
    got = engine.device_cos(x)
    want = _run(host_lib().libm_cos, x)
    same = got.view(np.uint64) == want.view(np.uint64)
    assert same.all(), (int((~same).sum()), x[~same][:5])
