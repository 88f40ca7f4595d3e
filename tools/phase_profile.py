"""Per-phase cycle profile of the specialised kernel (CTA 0): run with
EMTB200_CG_PROF=1 (and EMTB200_CG_DUMP=1 for the matching schedule dump).

    EMTB200_CG_PROF=1 python tools/phase_profile.py [workload] [steps] [warps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
warps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n = bench.WORKLOADS[wl][2]
b, _ = bench.build_batch(n, workload=wl)
e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, warps=warps,
                  tensor_solve=os.environ.get("TENSOR") == "1")
e.reserve(steps)
e.advance(steps, sync=True)
p = e.profile().astype(np.float64) / steps
G = int(e.summary.split("warps=")[1].split()[0])
used = np.nonzero(p[:G].sum(axis=0))[0]
print(e.summary[:200])
print("cycles per pass, CTA 0; rows = markers (even: phase compute, odd: barrier wait), cols = warps")
for m in used:
    row = p[:G, m]
    kind = "compute" if m % 2 == 0 else "wait   "
    print(f"m{m:02d} {kind} max {row.max():7.0f} min {row.min():7.0f} | " + " ".join(f"{x:6.0f}" for x in row))
tot = p[:G].sum(axis=1)
print(f"total per warp: " + " ".join(f"{x:6.0f}" for x in tot))
