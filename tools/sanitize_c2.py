import sys
sys.path.insert(0, ".")
import bench
from paper_1903_01081_b200 import engine
for wl in ("c2",):
    b, _ = bench.build_batch(1, workload=wl)
    e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
    e.reserve(60)
    e.advance(60, sync=True)
    print(wl, e.summary[:60], flush=True)
