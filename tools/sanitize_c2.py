"""C2 (single scenario, solo form) under compute-sanitizer: several short launches
with an L2-flush kernel on the engine stream between them (the bench's timing
pattern), then parity against the reference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import parity, ref  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

launches, per = int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 40
b, _ = bench.build_batch(1, workload="c2")
e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
e.reserve(launches * per)
stream = torch.cuda.ExternalStream(e.stream_ptr(), device=0)
buf = torch.zeros(16 * 1024 * 1024, dtype=torch.float32, device=0)
for k in range(launches):
    with torch.cuda.stream(stream):
        buf.add_(1.0)
    e.advance(per)
e.sync()
want = ref.execute(b.text(), b.initial, launches * per)
rep = parity.merge([parity.compare(e.waves().values, want.waves)])
print("c2", e.summary[:60], rep["bitwise_fraction"], rep.get("first_diff"), flush=True)
