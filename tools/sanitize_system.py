import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import bench
from conftest import GOLDEN_CASES, load_golden
from paper_1903_01081_b200 import engine
s, st = bench.load_scale_case(32)
e = engine.Engine(s, st, kernel=engine.KERNEL_SYSTEM)
e.reserve(3); e.advance(3, sync=True); print("scale32 ok", flush=True)
for name in GOLDEN_CASES:
    g = load_golden(name)
    try:
        engine.interpret(g.schedule, g.initial, min(g.steps, 50), kernel=engine.KERNEL_SYSTEM)
    except engine.EmtError as ex:
        print(name, "error (expected for error goldens):", ex.status)
print("done", flush=True)
