"""Cold-start end-to-end time of one bench step through the public API, JIT included.

    EMTB200_CACHE=<empty dir> python tools/cold_start.py <workload> <scenarios> <emt_steps> [device]

Runs in a fresh process (empty in-memory cubin cache) with an empty on-disk cache:
engine creation (schedule parse, code generation, NVRTC compile, module load) +
the batch's H2D from pinned host memory + `emt_steps` passes + the waveform D2H.
Prints one JSON object (seconds). Called by bench.py for the `e2e_cold` key.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    wl, n, S = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    dev = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    import numpy as np
    import torch
    import bench
    from paper_1903_01081_b200 import engine
    torch.cuda.init()
    torch.zeros(1, device=dev)  # CUDA context outside the clock (the driver's, not ours)
    engine.lib()
    batch, info = bench.build_batch(n, workload=wl)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    ct, init = pin(batch.const_table), pin(batch.initial)
    out = torch.empty((S, len(info.channels) * batch.width), dtype=torch.float64, pin_memory=True).numpy()
    t0 = time.perf_counter()
    eng = engine.Engine(batch.schedule, init, const_table=ct, width=batch.width, device=dev)
    t1 = time.perf_counter()
    eng.run(S, out, chunk=min(S, 1000))
    t2 = time.perf_counter()
    summ = eng.summary
    jit = float(summ.split("jit=")[1].split("s")[0]) if "jit=" in summ else None
    print(json.dumps({"create_s": t1 - t0, "run_s": t2 - t1, "total_s": t2 - t0, "jit_s": jit,
                      "cached": "(cached)" in summ, "kernel": summ[:120]}))


if __name__ == "__main__":
    main()
