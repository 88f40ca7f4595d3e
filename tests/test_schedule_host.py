"""Host-side helpers: text formats, N-1 widening, case generator."""
import json

import numpy as np

from conftest import bitwise_equal, load_golden
from oracle import oracle
from paper_1903_01081_b200 import cases
from paper_1903_01081_b200 import schedule as sch


def test_state_roundtrip():
    g = load_golden("feeder_w4")
    text = sch.format_state(g.initial, g.initial.size // g.width, g.width)
    back, w = sch.parse_state(text)
    assert w == g.width and bitwise_equal(back, g.initial)


def test_widen_width1_is_identity_for_oracle():
    g = load_golden("ieee39")
    info = sch.parse_info(g.schedule)
    text = sch.widen_text(g.schedule, info.const_table)
    a = oracle.Schedule(g.schedule).interpret(g.initial, 50)
    b = oracle.Schedule(text).interpret(g.initial, 50)
    assert bitwise_equal(a.waves, b.waves)


def test_n1_batch_lanes_equal_single_runs():
    """Lane s of the widened batch == the width-1 run with only that breaker's time changed."""
    g = load_golden("ieee39")
    info = sch.parse_info(g.schedule)
    ids = [c["id"] for c in json.loads(cases.ieee39_document())["components"]]
    scen = [("sw03", 0.002), ("sw40", 0.0031), ("sw17", 0.0042)]
    batch = sch.n1_batch(g.schedule, g.initial, ids, scen)
    wide = oracle.Schedule(batch.text()).interpret(batch.initial, 120)
    order = {c: i for i, c in enumerate(sorted(ids))}
    slots = sch.switch_toggle_slots(info)
    for lane, (sw, tf) in enumerate(scen):
        ct = info.const_table.copy()
        ct[slots[order[sw]], 0] = tf
        single = oracle.Schedule(sch.widen_text(g.schedule, ct)).interpret(g.initial, 120)
        cols = [c * 3 + lane for c in range(info.channels.__len__())]
        assert bitwise_equal(wide.waves[:, cols], single.waves)
    assert wide.factor_count == 1 + 3


def test_ieee39_document_shape():
    doc = json.loads(cases.ieee39_document())
    kinds = {}
    for c in doc["components"]:
        kinds[c["kind"]] = kinds.get(c["kind"], 0) + 1
    assert kinds["switch"] == 46 and kinds["voltage_source"] == 10
    assert kinds["series_rl"] == 46 + 19
    assert len(doc["nodes"]) == 39 + 46
    assert len(cases.n1_scenarios(1000)) == 1000
    assert cases.n1_scenarios(1000)[23] == (1, 0.10 + 0.01)


def _feeder_case():
    import gzip
    import os
    d = os.path.join(os.path.dirname(sch.__file__), "data")
    s = gzip.open(os.path.join(d, "feeder33_pv3.cgmsched.gz"), "rt").read()
    st, _ = sch.parse_state(gzip.open(os.path.join(d, "feeder33_pv3.state.gz"), "rt").read())
    meta = json.load(open(os.path.join(d, "feeder33_pv3.json")))
    return s, st, meta


def test_pv_sweep_batch_equals_reference_vectorize():
    """The C5 shared-G widening == the reference's own vectorize of gen_scenarios rows, bit for bit."""
    import pytest
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    s, st, meta = _feeder_case()
    pvm = meta["pv_sweep"]
    scen = sch.pv_grid(3, 2)
    batch = sch.pv_sweep_batch(s, st, pvm, scen)
    doc = open("/root/reference/proj/data/feeder33_pv3.json").read() if __import__("os").path.exists(
        "/root/reference/proj/data/feeder33_pv3.json") else None
    if doc is None:
        pytest.skip("reference document not present (GPU box)")
    rows = [[o for pv in pvm["pvs"] for o in ({"component": pv, "param": "irradiance", "value": irr},
                                               {"component": pv, "param": "temperature", "value": tmp})]
            for irr, tmp in scen]
    c = ref.compile_document(doc, rows=rows)
    info = sch.parse_info(c.schedule)
    assert bitwise_equal(info.const_table, batch.const_table)
    assert bitwise_equal(ref.parse_state(c.state), batch.initial)
    # and the executor agrees on the widened batch
    a = ref.execute(batch.text(), batch.initial, 300)
    b = oracle.Schedule(batch.text()).interpret(batch.initial, 300)
    assert bitwise_equal(a.waves, b.waves)


def test_pv_sweep_g_is_lane_invariant():
    """Every matrix-term conductance of the C5 batch is lane-invariant (shared G)."""
    s, st, meta = _feeder_case()
    batch = sch.pv_sweep_batch(s, st, meta["pv_sweep"], sch.pv_grid(4, 4))
    ct = batch.const_table
    varying = {k for k in range(ct.shape[0]) if not np.all(ct[k] == ct[k, 0])}
    assert varying == set(meta["pv_sweep"]["const_slots"])
    assert len(sch.pv_grid()) == 4096
