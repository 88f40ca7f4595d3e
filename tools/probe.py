"""Quick device timing probe (not the bench contract): engine step rate on the data cases."""
import gzip
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_01081_b200 import cases, engine  # noqa: E402
from paper_1903_01081_b200 import schedule as sch  # noqa: E402

DATA = os.path.join(ROOT, "paper_1903_01081_b200", "data")


def load(name):
    s = gzip.open(os.path.join(DATA, f"{name}.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(DATA, f"{name}.state.gz"), "rt").read())
    ids = json.load(open(os.path.join(DATA, f"{name}.json")))["component_ids"]
    return s, st, ids


def run(label, schedule, initial, const_table=None, width=0, steps=2000, lpb=0, kernel=0, warps=0):
    t0 = time.perf_counter()
    eng = engine.Engine(schedule, initial, const_table=const_table, width=width, lanes_per_block=lpb, kernel=kernel,
                        warps=warps)
    tc = time.perf_counter() - t0
    eng.reserve(steps + 200)
    eng.advance(200, sync=True)
    t = time.perf_counter()
    eng.advance(steps, sync=True)
    dt = time.perf_counter() - t
    W = eng.lanes
    print(f"{label:40s} W={W:5d} {dt / steps * 1e6:8.3f} us/step  {W * steps / dt:.3e} scen-steps/s  "
          f"fc={eng.stats().factor_count} create={tc:.2f}s | {eng.summary[:150]}", flush=True)
    return eng


def main():
    s, st, ids = load("ieee39")
    run("ieee39 W=1 generic", s, st, kernel=2)
    for w in (2, 4, 8):
        run(f"ieee39 W=1 spec warps={w}", s, st, warps=w)
    scen = cases.n1_scenarios(1000)
    b = sch.n1_batch(s, st, ids, [(f"sw{br:02d}", tf) for br, tf in scen])
    run("ieee39 N-1 W=1000 generic", s, b.initial, b.const_table, b.width, kernel=2, lpb=8)
    for w in (2, 4, 8, 16):
        run(f"ieee39 N-1 W=1000 spec warps={w}", s, b.initial, b.const_table, b.width, warps=w)
    f, fst, _ = load("feeder33_pv3")
    run("feeder W=1 generic", f, fst, kernel=2)
    run("feeder W=1 spec", f, fst)
    info = sch.parse_info(f)
    for W in (1000, 4096):
        ct = np.repeat(info.const_table, W, axis=1)
        init = np.repeat(fst.reshape(-1, 1), W, axis=1).reshape(-1)
        for w in (4, 8):
            run(f"feeder W={W} spec warps={w}", f, init, ct, W, warps=w)


if __name__ == "__main__":
    main()
