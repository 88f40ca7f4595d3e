"""Where the e2e time goes: replays bench.py's two-engine e2e pipeline for C3 and
records CUDA events on each engine's stream around commit and around the run, so
the GPU-side span of every batch can be set against host wall time per batch.

    python tools/e2e_probe.py [steps] [chunk]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1903_01081_b200 import engine  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 334
S = 1000
batch, info = bench.build_batch(1000, workload="c3")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
ct_host, init_host = pin(batch.const_table), pin(batch.initial)
bufs = [torch.empty((S, len(info.channels) * batch.width), dtype=torch.float64, pin_memory=True).numpy()
        for _ in range(2)]
engs = [engine.Engine(batch.schedule, init_host, const_table=ct_host, width=batch.width) for _ in range(2)]
streams = [torch.cuda.ExternalStream(x.stream_ptr()) for x in engs]
for x in engs:
    x.reserve(S)


def run(n, evs=None):
    done = [None, None]
    engs[0].stage(init_host, ct_host)
    for k in range(n):
        E, O = k % 2, (k + 1) % 2
        if k >= 2:
            engs[E].wait()
        if done[O] is not None:
            streams[E].wait_event(done[O])
        if evs is not None:
            evs[k][0].record(streams[E])
        engs[E].commit()
        if evs is not None:
            evs[k][1].record(streams[E])
        if k + 1 < n:
            engs[O].stage(init_host, ct_host)
        engs[E].run_async(S, bufs[E], chunk=chunk)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(streams[E])
        done[E] = ev
        if evs is not None:
            evs[k][2] = ev
    for x in engs:
        x.wait()


run(2)
torch.cuda.synchronize()
evs = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), None] for _ in range(steps)]
t0 = time.perf_counter()
run(steps, evs)
wall = (time.perf_counter() - t0) / steps * 1e3
torch.cuda.synchronize()
commit = [a.elapsed_time(b) for a, b, _ in evs]
runms = [b.elapsed_time(c) for _, b, c in evs]
span = evs[0][0].elapsed_time(evs[-1][2]) / steps
gaps = [evs[k][2].elapsed_time(evs[k + 1][0]) for k in range(steps - 1)]
print(f"wall/batch {wall:.3f} ms; GPU span/batch {span:.3f} ms")
print("commit ms", " ".join(f"{x:.3f}" for x in commit))
print("run ms   ", " ".join(f"{x:.3f}" for x in runms))
print("gap ms   ", " ".join(f"{x:.3f}" for x in gaps))
# the same batches without H2D/D2H: reload (untimed), then time the 1000 passes alone
e = engs[0]
dev_ms = []
for _ in range(steps):
    e.load(init_host, ct_host)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(streams[0])
    e.advance(S)
    b.record(streams[0])
    torch.cuda.synchronize()
    dev_ms.append(a.elapsed_time(b))
print("device-only advance ms", " ".join(f"{x:.3f}" for x in dev_ms))
