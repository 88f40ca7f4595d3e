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


def run(label, schedule, initial, const_table=None, width=0, steps=2000, lpb=0):
    eng = engine.Engine(schedule, initial, const_table=const_table, width=width, lanes_per_block=lpb)
    eng.reserve(steps + 200)
    eng.advance(200, sync=True)
    t = time.perf_counter()
    eng.advance(steps, sync=True)
    dt = time.perf_counter() - t
    W = eng.lanes
    print(f"{label:40s} W={W:5d} {dt / steps * 1e6:8.3f} us/step  {W * steps / dt:.3e} scen-steps/s  "
          f"fc={eng.stats().factor_count}", flush=True)
    return eng


def main():
    s, st, ids = load("ieee39")
    run("ieee39 W=1", s, st)
    scen = cases.n1_scenarios(1000)
    b = sch.n1_batch(s, st, ids, [(f"sw{br:02d}", tf) for br, tf in scen])
    for lpb in (0, 1, 2, 4, 8):
        run(f"ieee39 N-1 W=1000 lpb={lpb}", s, b.initial, b.const_table, b.width, lpb=lpb)
    f, fst, _ = load("feeder33_pv3")
    run("feeder W=1", f, fst)
    info = sch.parse_info(f)
    for W in (1000, 4096):
        ct = np.repeat(info.const_table, W, axis=1)
        init = np.repeat(fst.reshape(-1, 1), W, axis=1).reshape(-1)
        run(f"feeder W={W}", f, init, ct, W)


if __name__ == "__main__":
    main()
