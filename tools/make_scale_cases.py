"""Compiles the reference's large single-system cases with the REAL reference.

    make -C oracle ref && python tools/make_scale_cases.py [k ...]

gen_scale_case(feeder33_pv3, k) (proj/src/bench.cpp:54-117: k copies of the
bundled feeder joined at its root node, the paper's large-scale test,
PAPER.md:139-147) -> parse_model -> compile_task (proj/src/pipeline.cpp:5-18).
Writes paper_1903_01081_b200/data/feeder_scale<k>.cgmsched.gz / .state.gz, the
executor's inputs, so the GPU box (no /root/reference) can run and bench them.
k = 32 and 128 are SURVEY §6's probe sizes; k = 330 is the paper's largest case
(990 PV subsystems, 77,220 control blocks).
"""
from __future__ import annotations

import gzip
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

DATA = os.path.join(ROOT, "paper_1903_01081_b200", "data")
FEEDER = "/root/reference/proj/data/feeder33_pv3.json"


def main(ks):
    doc = open(FEEDER).read()
    for k in ks:
        t0 = time.time()
        c = ref.compile_document(ref.gen_scale_case(doc, k))
        for ext, text in (("cgmsched", c.schedule), ("state", c.state)):
            with gzip.open(os.path.join(DATA, f"feeder_scale{k}.{ext}.gz"), "wt", compresslevel=9) as f:
                f.write(text)
        print(f"k={k}: {c.schedule.splitlines()[1]} ({time.time() - t0:.1f} s)")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [32, 128])
