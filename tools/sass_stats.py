"""SASS statistics of a generated step-loop kernel, without a GPU.

    python tools/sass_stats.py [c3|c2|c5|c4] [--keep DIR]

Generates the kernel source for the workload (engine.codegen, same options as
the engine), compiles it with nvcc for sm_100a (-fmad=false, like jit.cpp) and
counts SASS instructions of emt_cg_kernel: total, FP64 ops, shared loads /
stores, barriers, branches, calls — the static side of an A/B before spending
GPU time."""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
    keep = sys.argv[sys.argv.index("--keep") + 1] if "--keep" in sys.argv else tempfile.mkdtemp()
    import bench
    from paper_1903_01081_b200 import engine
    n = {"c3": 1000, "c2": 1, "c5": 4096, "c4": 120}[wl]
    b, _ = bench.build_batch(n, workload=wl)
    src, summary = engine.codegen(b.schedule, b.const_table, b.width, warps=8, compile=False)
    cu = os.path.join(keep, f"{wl}.cu")
    open(cu, "w").write(src)
    cubin = cu[:-3] + ".cubin"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-fmad=false",
                           "-std=c++17", "-w", "-o", cubin, cu])
    sass = subprocess.check_output(["cuobjdump", "-sass", "-fun", "emt_cg_kernel", cubin], text=True)
    ops = collections.Counter()
    for ln in sass.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
        if m:
            ops[m.group(2).split(".")[0]] += 1
    total = sum(ops.values())
    print(f"{wl}: {summary[:90]}")
    print(f"emt_cg_kernel SASS: {total} instructions")
    for k in ("DFMA", "DADD", "DMUL", "DSETP", "LDS", "STS", "LDG", "STG", "BAR", "BRA", "CALL", "MUFU"):
        print(f"  {k:6s} {ops.get(k, 0)}")


if __name__ == "__main__":
    main()
