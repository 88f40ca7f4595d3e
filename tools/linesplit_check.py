"""Multi-process check of the device-side line exchange (CUDA IPC mirror + progress):
each rank owns a lane shard of the C4 system, rank 0 compares the gathered
waveforms with a single-engine run bit for bit.

    BENCH_SHARE_GPU=1 python -m torch.distributed.run --nproc-per-node 2 tools/linesplit_check.py [host|device]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
from paper_1903_01081_b200 import engine, sharding  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "device"
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = 0 if os.environ.get("BENCH_SHARE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(dev)
W, steps = 64, 700
b, _ = bench.build_batch(W, workload="c4")
lo, hi = sharding.shard_bounds(W, world, rank)
sh = sharding.LineSplitShard(dist, b, lo, hi, device=dev, exchange=mode)
sh.eng.reserve(steps + 200)
sh.advance(steps)
sh.eng.sync()
import time
dist.barrier()
t0 = time.perf_counter()
sh.advance(200)
sh.eng.sync()
dt = (time.perf_counter() - t0) / 200
if rank == 0:
    print(f"linesplit {mode} {os.environ.get('EMTB200_LINE_SCOPE', 'sys')}: {dt * 1e6:.2f} us/pass", flush=True)
sh.eng.reserve(steps)
sh.reload(b.initial, b.const_table)
sh.advance(steps)
sh.eng.sync()
got = torch.from_numpy(sh.eng.waves().values.copy())
parts = [torch.zeros((steps, 5 * (b_ - a_)), dtype=torch.float64)
         for a_, b_ in (sharding.shard_bounds(W, world, r) for r in range(world))]
dist.gather(got, parts if rank == 0 else None, dst=0) if hasattr(dist, "gather") else None
if rank == 0:
    whole = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=W)
    whole.reserve(steps)
    whole.advance(steps)
    want = whole.waves().values
    ok = True
    for r, part in enumerate(parts):
        a_, b_ = sharding.shard_bounds(W, world, r)
        n = b_ - a_
        for c in range(5):
            ok &= bool((part.numpy()[:, c * n:(c + 1) * n].view(np.uint64) == want[:, c * W + a_:c * W + b_].view(np.uint64)).all())
    print(f"linesplit {mode} world={world}: bitwise {'OK' if ok else 'MISMATCH'}; launches={sh.eng.stats().kernel_launches}", flush=True)
dist.destroy_process_group()
