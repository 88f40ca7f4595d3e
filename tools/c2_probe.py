"""Diagnose a C2 (single scenario) parity difference: the same engine run with
and without an L2-flush write between launches, against the reference."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import parity, ref  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = {"c2": 1, "c3": 1000}[wl]
batch, info = bench.build_batch(n, workload=wl)
steps = 23000
want = ref.execute(batch.text(), batch.initial, steps)
for flush in (False, True):
    eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width)
    eng.reserve(steps)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=0)
    buf = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=0)
    for k in range(23):
        if flush:
            with torch.cuda.stream(stream):
                buf.add_(1.0)
        eng.advance(1000)
    eng.sync()
    rep = parity.merge([parity.compare(eng.waves(0, steps).values, want.waves)])
    print(wl, "flush" if flush else "noflush", eng.summary[:60], {k: rep[k] for k in ("bitwise_fraction", "fail", "max_abs_diff")},
          rep.get("first_diff"))
