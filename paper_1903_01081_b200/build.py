"""In-tree build of libemtb200.so for sm_100a (nvcc cross-compiles without a GPU).

The shared object is written next to this file so that it travels with the
repository snapshot to the GPU box; nothing is JIT-compiled at import time.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libemtb200.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("engine.cu", "host_schedule.cpp", "codegen.cpp", "emit_program.cpp", "jit.cpp", "waveform_text.cpp")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in ("host_schedule.hpp", "codegen.hpp", "jit.hpp", "libmcos.cuh", "system_kernel.cuh")] + [
    os.path.join(ROOT, "include", "emt_b200.h")]
CUDA = "/usr/local/cuda"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo",
    "-fmad=false",            # no FMA contraction: the reference builds with -ffp-contract=off
    "-std=c++17",
    "-ccbin", "/usr/bin/g++",  # system libstdc++ (dynamic), same as the Python process
    "-Xcompiler", "-fPIC", "-shared",
    # NVRTC (runtime code generation); driver entry points come via cudaGetDriverEntryPoint
    f"-L{CUDA}/lib64", "-lnvrtc", f"-Xlinker=-rpath,{CUDA}/lib64",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


FLAVOUR = LIB + ".flavour"  # "dev" or "product": the build the library was made as


def stale(dev: bool = False) -> bool:
    if not os.path.exists(LIB):
        return True
    try:
        with open(FLAVOUR) as f:
            if f.read().strip() != ("dev" if dev else "product"):
                return True  # a product build after a dev build (or the reverse) recompiles
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, dev: bool = False) -> str:
    """dev=True: a developer build whose generator reads EMTB200_CG_* A/B knobs from the
    environment (the product build ignores the environment; bench.py refuses a dev build)."""
    if not force and not stale(dev):
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DEMTB200_DEV_KNOBS"] if dev else []), "-o", LIB, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    with open(FLAVOUR, "w") as f:
        f.write("dev" if dev else "product")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv or "--dev" in sys.argv, verbose=True, dev="--dev" in sys.argv)
    print(LIB)
