"""Accuracy of the shared-G tensor-core solve vs the exact LU path (C5 PV grid):
max |a-b| relative to each channel's amplitude, and how many samples miss the
strict per-sample bar |a-b| <= 1e-12 + 1e-9|b|. Writes profiles/dmma_accuracy_<tag>.json."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

lanes, steps = int(sys.argv[1]) if len(sys.argv) > 1 else 256, int(sys.argv[2]) if len(sys.argv) > 2 else 20000
b, _ = bench.build_batch(lanes, workload="c5")
out = {}
for ts in (False, True):
    e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width, tensor_solve=ts)
    e.reserve(steps)
    e.advance(steps)
    out[ts] = (e.waves().values, e.summary)
exact, dm = out[False][0], out[True][0]
amp = np.abs(exact).max(axis=0)
err = np.abs(dm - exact)
rel_amp = float((err / np.maximum(amp, 1e-300)).max())
strict_bad = int(np.sum(err > 1e-12 + 1e-9 * np.abs(exact)))
res = {"lanes": lanes, "steps": steps, "samples": int(exact.size), "max_abs_err": float(err.max()),
       "max_err_over_channel_amplitude": rel_amp, "samples_missing_strict_bar": strict_bad,
       "strict_bar": "|a-b| <= 1e-12 + 1e-9|b| per sample", "kernel": out[True][1][:160]}
print(json.dumps(res))
json.dump(res, open(f"gpurun_out/dmma_accuracy.json", "w"), indent=1)
