"""The `transmission_line` document kind (EXTENSION — the reference
has no line model): validation mirrors the reference's check_component
(proj/src/model.cpp:154-222), and a document that declares a line compiles (the
reference's own parse_model -> compile_task) and runs bit-identically to the same
system written with the placeholder line ends by hand (lines.add_line_end).
"""
import json

import numpy as np
import pytest

from conftest import bitwise_equal
from oracle import oracle, ref
from paper_1903_01081_b200 import lines

DT = 50e-6


def line_doc(zc=400.0, tau=10 * DT, load=0.0, **extra):
    d = json.loads(lines.single_line_document(zc=zc, load=load))
    d["components"] = [c for c in d["components"] if not c["id"].startswith(("la_", "lb_"))]
    c = {"id": "l", "kind": "transmission_line", "terminals": ["a", "b"],
         "params": {"surge_impedance": zc, "travel_time": tau}}
    c.update(extra)
    d["components"].append(c)
    return json.dumps(d)


def reference_compile(document):
    c = ref.compile_document(document)
    return c.schedule, ref.parse_state(c.state)


@pytest.mark.parametrize("mutate,code", [
    (lambda c: c["params"].pop("travel_time"), "InvalidParameter"),
    (lambda c: c["params"].__setitem__("surge_impedance", -1.0), "InvalidParameter"),
    (lambda c: c["params"].__setitem__("surge_impedance", float("inf")), "InvalidParameter"),
    (lambda c: c["params"].__setitem__("length", 3.0), "InvalidParameter"),
    (lambda c: c["params"].__setitem__("travel_time", 1.5 * DT), "InvalidParameter"),
    (lambda c: c.__setitem__("terminals", ["a"]), "InvalidParameter"),
    (lambda c: c.__setitem__("terminals", ["a", "a"]), "InvalidParameter"),
    (lambda c: c.__setitem__("terminals", ["a", "0"]), "InvalidParameter"),
    (lambda c: c.__setitem__("terminals", ["a", "nowhere"]), "DanglingReference"),
    (lambda c: c.__setitem__("id", "src"), "DuplicateIdentifier"),
])
def test_validation_mirrors_check_component(mutate, code):
    d = json.loads(line_doc())
    mutate(d["components"][-1])
    with pytest.raises(lines.LineDocumentError) as ei:
        lines.expand_document(json.dumps(d))
    assert ei.value.code == code


def test_expansion_stamps_two_coupled_ends():
    doc, spec = lines.expand_document(line_doc(zc=300.0, tau=7.5 * DT))
    ids = [c["id"] for c in json.loads(doc)["components"]]
    assert {"l__a_h", "l__a_z", "l__b_h", "l__b_z"} <= set(ids)
    assert spec.ends == ["l__a", "l__b"] and spec.zc == [300.0, 300.0]
    assert spec.peers.tolist() == [[[0, 1], [0, 0]]]
    lines.check_symmetric(spec)


@pytest.mark.skipif(not ref.available(), reason="needs oracle/_ref (make -C oracle ref)")
@pytest.mark.parametrize("load", [0.0, 400.0, 1000.0])
def test_document_line_equals_hand_written_placeholders(load):
    tau = 10 * DT
    got = lines.document_batch(line_doc(tau=tau, load=load), reference_compile)
    hand_doc = lines.single_line_document(load=load)
    s, st = reference_compile(hand_doc)
    ids = [c["id"] for c in json.loads(hand_doc)["components"]]
    want = lines.bergeron_batch(s, st, ids, lines.single_line_spec(400.0, tau))
    a = oracle.Schedule(got.text()).interpret(got.initial, 200).waves
    b = oracle.Schedule(want.text()).interpret(want.initial, 200).waves
    assert bitwise_equal(a, b)
    if load == 0.0:  # open end: the far bus sees 2 x the incident E/2 after one travel time
        np.testing.assert_allclose(a[10:, 1], 1000.0, rtol=1e-12)


@pytest.mark.skipif(not ref.available(), reason="needs oracle/_ref (make -C oracle ref)")
def test_document_without_lines_passes_through():
    doc = json.loads(line_doc())
    doc["components"] = [c for c in doc["components"] if c["kind"] != "transmission_line"]
    doc["components"].append({"id": "rl", "kind": "resistor", "params": {"resistance": 10.0}, "terminals": ["b", "0"]})
    doc["components"].append({"id": "rab", "kind": "resistor", "params": {"resistance": 5.0}, "terminals": ["a", "b"]})
    b = lines.document_batch(json.dumps(doc), reference_compile)
    s, st = reference_compile(json.dumps(doc))
    assert b.schedule == s and bitwise_equal(b.initial, st)
