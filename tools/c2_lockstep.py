"""Find the first arena slot that goes wrong in a C2 run perturbed by an L2-flush
kernel between launches: two engines in lockstep (one perturbed), arenas compared
after every launch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
per = int(sys.argv[2]) if len(sys.argv) > 2 else 50
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 400
n = {"c2": 1, "c3": 64}[wl]
b, info = bench.build_batch(n, workload=wl)
ea = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
eb = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
for e in (ea, eb):
    e.reserve(per * nl)
stream = torch.cuda.ExternalStream(eb.stream_ptr(), device=0)
buf = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=0)
mat = next(ln for ln in b.schedule.splitlines() if ln.startswith("MATRIX"))
print(mat, flush=True)
for k in range(nl):
    ea.advance(per)
    with torch.cuda.stream(stream):
        buf.add_(1.0)
    eb.advance(per)
    ea.sync(); eb.sync()
    sa, sb = ea.state(), eb.state()
    if not np.array_equal(sa.view(np.uint64), sb.view(np.uint64)):
        d = np.nonzero(sa.view(np.uint64) != sb.view(np.uint64))[0]
        ext = sa.size // b.width
        print("launch", k, "differing slots", sorted(set((d // b.width).tolist()))[:40], "count", d.size, flush=True)
        wa, wb = ea.waves(k * per, per).values, eb.waves(k * per, per).values
        rows = np.nonzero((wa != wb).any(1))[0]
        print("first differing row within launch", rows[:5], flush=True)
        break
else:
    print("no difference over", nl, "launches", flush=True)
