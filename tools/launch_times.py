"""Per-launch device times of the C3 sweep (1000 passes per launch): refactorisation
cost shows up in the launches that contain fault times (0.10-0.31 s = passes 2000-6200)."""
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_1903_01081_b200 import engine
b, _ = bench.build_batch(1000)
e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
e.reserve(12000)
s = torch.cuda.ExternalStream(e.stream_ptr())
out = []
for k in range(12):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    e.advance(1000)
    t1.record(s)
    e.sync()
    out.append(t0.elapsed_time(t1))
print("ms per 1000 passes:", " ".join(f"{x:.3f}" for x in out))
print("refactor passes:", len(e.refactor_steps()))
