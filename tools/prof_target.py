"""Small profiling target: one engine launch of the N-1 batch (for ncu).

    python tools/prof_target.py [--lanes 1000] [--steps 200] [--warps 8] [--kernel 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lanes", type=int, default=1000)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--warps", type=int, default=8)
ap.add_argument("--kernel", type=int, default=1)
ap.add_argument("--dump", default="")
a = ap.parse_args()
batch, info = bench.build_batch(a.lanes)
eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width,
                    kernel=a.kernel, warps=a.warps)
print(eng.summary, flush=True)
if a.dump:
    open(a.dump, "w").write(eng.source)
eng.reserve(3 * a.steps)
eng.advance(a.steps, sync=True)  # warm-up launch (includes the first refactorisation)
eng.advance(a.steps, sync=True)
eng.advance(a.steps, sync=True)
print("ok", eng.stats())
