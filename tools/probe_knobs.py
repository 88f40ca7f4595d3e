"""A/B timing of code-generator knobs on the N-1 batch (dev tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_1903_01081_b200 import engine

batch, info = bench.build_batch(int(os.environ.get("LANES", "1000")))
for spec in sys.argv[1:]:
    env = dict(kv.split("=") for kv in spec.split(",") if "=" in kv)
    for k, v in env.items():
        os.environ[k] = v
    warps = int(env.get("WARPS", "8"))
    eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width, warps=warps,
                        kernel=int(env.get("KERNEL", "0")))
    eng.reserve(2200)
    eng.advance(200, sync=True)
    t = time.perf_counter()
    eng.advance(2000, sync=True)
    dt = time.perf_counter() - t
    print(f"{spec:50s} {dt / 2000 * 1e6:7.3f} us/step {batch.width * 2000 / dt:.3e} | {eng.summary[:120]}", flush=True)
    for k in env:
        os.environ.pop(k, None)
