"""One C3 launch of a single pass (for profiling the per-launch prologue/epilogue)."""
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

b, info = bench.build_batch(1000, workload="c3")
e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
e.reserve(100)
for _ in range(4):
    e.advance(1, sync=True)
