"""Dev-build check (build.py --dev, EMTB200_CG_POISON=1): shared memory is NaN at
kernel entry, so a slot read before the launch writes it breaks parity at once."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import parity, ref  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

for wl, n, steps, per in (("c2", 1, 3000, 1000), ("c3", 64, 3000, 1000), ("c5", 64, 2000, 500), ("c4", 8, 2000, 500)):
    b, _ = bench.build_batch(n, workload=wl)
    e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
    e.reserve(steps)
    for _ in range(steps // per):
        e.advance(per)
    e.sync()
    if wl == "c4":
        from oracle import oracle
        want = oracle.Schedule(b.text()).interpret(b.initial, steps).waves
    else:
        want = ref.execute(b.text(), b.initial, steps).waves
    rep = parity.merge([parity.compare(e.waves().values, want)])
    print(wl, e.summary[-60:], rep["bitwise_fraction"], rep.get("first_diff"), flush=True)
