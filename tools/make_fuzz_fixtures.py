"""Property-style parity set: seeded random documents (tests/golden/docs.py:fuzz)
compiled and run by the REAL reference (compile_task + interpret), stored as
tests/golden/fuzz/fuzz_<seed>.{cgmsched.gz,state.gz,npz} (waves, time,
factor_count, or the reference's error code and message).

    make -C oracle ref && python tools/make_fuzz_fixtures.py [count]
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


def main(count):
    os.makedirs(OUT, exist_ok=True)
    for seed in range(count):
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


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
