import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_1903_01081_b200 import engine
b, info = bench.build_batch(1000, workload="c3")
e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
e.reserve(20000)
st = torch.cuda.ExternalStream(e.stream_ptr())
e.advance(100, sync=True)
def t(n, reps):
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(reps):
        e.advance(n)
    c.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(c) / reps
for n in (1, 2, 10, 100):
    print(n, f"{t(n, 50 if n < 100 else 10) * 1e3:.1f} us per launch")
