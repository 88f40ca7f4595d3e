"""Cold-start end-to-end time of one bench step through the public API, JIT included.

    python tools/cold_start.py <workload> <scenarios> <emt_steps> <device> <sync|async>

Runs in a fresh process (empty in-memory cubin cache) with an empty on-disk cache:
engine creation + the batch's H2D from pinned host memory + `emt_steps` passes +
the waveform D2H, either with the JIT before the first pass (`sync`) or with
EMT_FLAG_ASYNC_JIT (`async`: the generic kernel runs while NVRTC compiles; the
engine switches to the specialised kernel when it is ready). Prints one JSON
object (seconds) and writes the waveform digest. Called twice by bench.py for
the `e2e_cold` key.
"""
import json
import os
import sys
import tempfile
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
    mode = sys.argv[5] if len(sys.argv) > 5 else "sync"
    cache = tempfile.TemporaryDirectory()  # empty on-disk cubin cache, removed at exit
    os.environ["EMTB200_CACHE"] = cache.name
    out = torch.empty((S, len(info.channels) * batch.width), dtype=torch.float64, pin_memory=True).numpy()
    t0 = time.perf_counter()
    eng = engine.Engine(batch.schedule, init, const_table=ct, width=batch.width, device=dev, async_jit=mode == "async")
    t1 = time.perf_counter()
    eng.run(S, out, chunk=min(S, 100 if mode == "async" else 1000))
    t2 = time.perf_counter()
    ran = eng.summary
    eng.wait_jit()
    summ = eng.summary
    jit = float(summ.split("jit=")[1].split("s")[0]) if "jit=" in summ else None
    import hashlib
    res = {"mode": mode, "total_s": t2 - t0, "create_s": t1 - t0, "run_s": t2 - t1, "jit_s": jit,
           "kernel_during_run": ran[:90], "digest": hashlib.sha1(out.tobytes()).hexdigest()}
    eng.close()
    print(json.dumps(res))
    cache.cleanup()


if __name__ == "__main__":
    main()
