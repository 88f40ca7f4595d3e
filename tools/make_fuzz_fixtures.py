"""Property-style parity set: seeded random documents (tests/golden/docs.py:fuzz)
compiled and run by the REAL reference (compile_task + interpret), stored as
tests/golden/fuzz/fuzz_<seed>.{cgmsched.gz,state.gz,npz} (waves, time,
factor_count, or the reference's error code and message).

    make -C oracle ref && python tools/make_fuzz_fixtures.py [count]
    python -c "import tools.make_fuzz_fixtures as m; m.main(64, start=24)"   # add seeds 24..63 only
"""
import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from oracle import ref  # noqa: E402
import docs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fuzz")


def main(count, start=0):
    os.makedirs(OUT, exist_ok=True)
    for seed in range(start, count):
        doc = docs.fuzz(seed)
        c = ref.compile_document(doc)
        steps = json.loads(doc)["task"]["duration"] / json.loads(doc)["task"]["dt"]
        steps = int(round(steps))
        for ext, text in (("cgmsched", c.schedule), ("state", c.state)):
            with gzip.open(os.path.join(OUT, f"fuzz_{seed}.{ext}.gz"), "wt", compresslevel=9) as f:
                f.write(text)
        init = ref.parse_state(c.state)
        meta = json.dumps({"steps": steps, "note": f"docs.fuzz({seed})"})
        try:
            r = ref.execute(c.schedule, init, steps)
            np.savez_compressed(os.path.join(OUT, f"fuzz_{seed}.npz"), waves=r.waves, time=r.time,
                                factor_count=r.factor_count, error_code=0, meta=meta)
            print(f"fuzz_{seed}: {r.waves.shape} factor_count={r.factor_count}")
        except ref.RefError as e:
            np.savez_compressed(os.path.join(OUT, f"fuzz_{seed}.npz"), waves=np.zeros((0, 0)), time=np.zeros(0),
                                factor_count=0, error_code=e.code, error_msg=e.msg, meta=meta)
            print(f"fuzz_{seed}: error {e.code} {e.msg[:60]}")


def batched(count):
    """Vectorised variants (the reference's own `vectorize`, compile_task with override
    rows): per lane, other resistances, source magnitudes and controlled-source gain."""
    rng = np.random.default_rng(77)
    for seed in range(count):
        doc = docs.fuzz(100 + seed)
        d = json.loads(doc)
        res = [c["id"] for c in d["components"] if c["kind"] == "resistor"][:3]
        src = [c for c in d["components"] if c["kind"] in ("voltage_source", "current_source")][:1]
        W = int(rng.integers(3, 9))
        rows = []
        for _ in range(W):
            row = [{"component": r, "param": "resistance", "value": float(rng.uniform(0.3, 6.0))} for r in res]
            row += [{"component": c["id"], "param": "magnitude", "value": float(rng.uniform(0.5, 50.0))} for c in src]
            row.append({"component": "act", "param": "gain", "value": float(rng.uniform(-0.05, 0.05))})
            rows.append(row)
        c = ref.compile_document(doc, rows=rows)
        steps = int(round(d["task"]["duration"] / d["task"]["dt"]))
        name = f"fuzzw_{seed}"
        for ext, text in (("cgmsched", c.schedule), ("state", c.state)):
            with gzip.open(os.path.join(OUT, f"{name}.{ext}.gz"), "wt", compresslevel=9) as f:
                f.write(text)
        init = ref.parse_state(c.state)
        r = ref.execute(c.schedule, init, steps)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), waves=r.waves, time=r.time,
                            factor_count=r.factor_count, error_code=0,
                            meta=json.dumps({"steps": steps, "note": f"docs.fuzz({100 + seed}) x {W} lanes"}))
        print(f"{name}: W={W} {r.waves.shape} factor_count={r.factor_count}")


def with_lines(count):
    """Random documents plus 1-3 `transmission_line` components (the document kind,
    lines.document_batch). The reference has no line model: these are checked
    device == C oracle, and the stored waves are the oracle's."""
    from oracle import oracle
    from paper_1903_01081_b200 import lines
    from paper_1903_01081_b200 import schedule as sch
    rng = np.random.default_rng(99)
    for seed in range(count):
        d = json.loads(docs.fuzz(200 + seed))
        nodes = d["nodes"]
        for q in range(int(rng.integers(1, 4))):
            a, b = rng.choice(len(nodes), size=2, replace=False)
            d["components"].append({"id": f"tl{q}", "kind": "transmission_line", "terminals": [nodes[a], nodes[b]],
                                    "params": {"surge_impedance": float(rng.uniform(50.0, 500.0)),
                                               "travel_time": float(rng.uniform(2.0, 9.0)) * d["task"]["dt"]}})
        doc = json.dumps(d)
        batch = lines.document_batch(doc, lambda x: (lambda c: (c.schedule, ref.parse_state(c.state)))(ref.compile_document(x)))
        steps = int(round(d["task"]["duration"] / d["task"]["dt"]))
        name = f"fuzzl_{seed}"
        ext_n = batch.initial.size // batch.width
        with gzip.open(os.path.join(OUT, f"{name}.cgmsched.gz"), "wt", compresslevel=9) as f:
            f.write(batch.text())
        with gzip.open(os.path.join(OUT, f"{name}.state.gz"), "wt", compresslevel=9) as f:
            f.write(sch.format_state(batch.initial, ext_n, batch.width))
        r = oracle.Schedule(batch.text()).interpret(batch.initial, steps)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), waves=r.waves,
                            time=(np.arange(steps) + 1) * d["task"]["dt"], factor_count=r.factor_count, error_code=0,
                            meta=json.dumps({"steps": steps, "note": f"docs.fuzz({200 + seed}) + lines (C oracle)"}))
        print(f"{name}: {r.waves.shape} factor_count={r.factor_count}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
    batched(8)
    with_lines(6)
