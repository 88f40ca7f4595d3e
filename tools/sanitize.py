"""Small runs of every kernel variant for compute-sanitizer (racecheck / memcheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

cases = [("c3", 64, {}), ("c5", 64, {}), ("c5", 64, {"tensor_solve": True}), ("c4", 40, {}), ("c2", 1, {})]
for wl, n, kw in cases:
    b, _ = bench.build_batch(n, workload=wl)
    for kern in (engine.KERNEL_AUTO, engine.KERNEL_GENERIC, engine.KERNEL_TSIMT, engine.KERNEL_SYSTEM):
        if kw and kern != engine.KERNEL_AUTO:
            continue
        e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, kernel=kern, **kw)
        e.reserve(60)
        e.advance(60, sync=True)
        print(wl, n, kern, kw, e.summary[:60], flush=True)

# the system kernel on the reference's large-scale case (k = 32: TMA ring, tiles, rounds,
# producer / consumer backward sweep), including its factorisation
s, st = bench.load_scale_case(32)
e = engine.Engine(s, st, kernel=engine.KERNEL_SYSTEM)
e.reserve(4)
e.advance(2)
e.advance(2, sync=True)
print("scale32", e.summary[:60], flush=True)
