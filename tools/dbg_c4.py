import sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import test_bergeron as tb
from paper_1903_01081_b200 import engine
b = tb.c4_case(40)
want = tb.run_oracle(b, 50).waves
print("oracle nonzero", np.count_nonzero(want))
for env in ({"EMTB200_CG_SWSLIM": "0"}, {"EMTB200_CG_SWSLIM": "1"}, {"EMTB200_LINE_PERSISTENT": "0"}, {"EMTB200_CG_STRAIGHT": "1", "EMTB200_CG_WARPMAJOR": "0"}):
    for k, v in env.items(): os.environ[k] = v
    e = engine.Engine(b.schedule, b.initial, const_table=b.const_table, width=b.width)
    e.reserve(50)
    try:
        e.advance(50, sync=True)
        w = e.waves().values
        print(env, "nonzero", np.count_nonzero(w), "maxerr", np.abs(w - want).max(), e.stats().kernel_launches)
    except Exception as ex:
        print(env, "ERR", ex)
    for k in env: del os.environ[k]
