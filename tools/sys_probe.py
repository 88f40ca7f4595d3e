"""Times the system kernel on gen_scale_case cases: python tools/sys_probe.py [k ...]
With a developer build and EMTB200_CG_PROF=1 it also prints the phase split."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_1903_01081_b200 import engine

for k in [int(a) for a in sys.argv[1:]] or [32, 128]:
    s, st = bench.load_scale_case(k)
    t0 = time.time()
    eng = engine.Engine(s, st)
    print(k, eng.summary, f"create {time.time()-t0:.2f}s", flush=True)
    n = 200 if k <= 128 else 50
    eng.reserve(3 * n + 1)
    t0 = time.time(); eng.advance(1, sync=True); t_first = time.time() - t0
    if os.environ.get("EMTB200_CG_PROF"):
        pf = eng.profile()[0]
        print(json.dumps({"k": k, "factor_setup": int(pf[12]), "factor_elim": int(pf[13]), "factor_urow": int(pf[14]),
                          "elim_steps": int(pf[15]), "cycles_per_step": float(pf[13]) / max(1, int(pf[15]))}), flush=True)
    eng.advance(n, sync=True)
    prof0 = eng.profile()[0, :12].copy() if os.environ.get("EMTB200_CG_PROF") else None
    t0 = time.time(); eng.advance(n, sync=True); dt = (time.time() - t0) / n
    out = {"k": k, "first_pass_s": round(t_first, 4), "us_per_step": round(dt * 1e6, 2)}
    if prof0 is not None:
        d = (eng.profile()[0, :12] - prof0) / n
        out["cycles_per_pass"] = dict(zip(["layers", "factor", "gather_fwd", "bwd", "finalize", "bwd_consumer_wait", "bwd_consumer_chain", "bwd_producer_wait", "fwd_tile", "fwd_products", "fwd_chains", "gather"], d.tolist()))
    print(json.dumps(out), flush=True)
