"""Small model documents (reference JSON schema) used for golden fixtures.

Each mirrors a behaviour the reference's own tests pin (cited per builder),
written fresh here; values differ where that costs nothing.
"""
from __future__ import annotations

import json

import numpy as np


def _doc(nodes, components, channels, dt, duration, control=(), couplings=()):
    return json.dumps({
        "nodes": list(nodes), "components": list(components), "control": list(control),
        "couplings": list(couplings),
        "task": {"dt": dt, "duration": duration, "channels": list(channels), "device_profile": "cpu-serial",
                 "strategy": "serial"},
    }, indent=1) + "\n"


def comp(cid, kind, params, a, b):
    return {"id": cid, "kind": kind, "params": params, "terminals": [a, b]}


def rc_discharge(r=1000.0, c=1e-6, v0=1.0, dt=1e-6, duration=5e-3):
    """RC discharge (proj/tests/support/oracles.hpp:137-152, test_exec.cpp:29-35)."""
    return _doc(["1"], [comp("r1", "resistor", {"resistance": r}, "1", "0"),
                        comp("c1", "capacitor", {"capacitance": c, "v0": v0}, "1", "0")], ["v:1"], dt, duration)


def switched_rc():
    """AC source, breaker closing then opening (test_exec.cpp:54-75): factor_count 3."""
    return _doc(["1", "2"], [
        comp("vs", "voltage_source", {"magnitude": 10.0, "frequency": 50.0, "phase": 0.0, "rs": 0.5}, "1", "0"),
        comp("sw", "switch", {"state": "open", "toggle_times": [0.0003, 0.0006]}, "1", "2"),
        comp("rl", "resistor", {"resistance": 5.0}, "2", "0"),
        comp("cl", "capacitor", {"capacitance": 1e-05}, "2", "0"),
    ], ["v:2", "i:sw"], 1e-4, 1e-3)


def switched_dc():
    """DC source + one toggle, batched over the load resistance (test_exec.cpp:243-274): factor_count 2."""
    return _doc(["1", "2"], [
        comp("vs", "voltage_source", {"magnitude": 10.0, "frequency": 0.0, "phase": 0.0, "rs": 0.5}, "1", "0"),
        comp("sw", "switch", {"state": "open", "toggle_times": [0.0004]}, "1", "2"),
        comp("rl", "resistor", {"resistance": 5.0}, "2", "0"),
        comp("cl", "capacitor", {"capacitance": 1e-05}, "2", "0"),
    ], ["v:2", "i:sw"], 1e-4, 1e-3)


def cyclic_controls():
    """Algebraic loop + integrator feedback through meter/actuator (test_exec.cpp:181-222)."""
    return _doc(["1"], [
        comp("r1", "resistor", {"resistance": 10.0}, "1", "0"),
        comp("is", "current_source", {"magnitude": 1.0, "frequency": 50.0, "phase": 0.0}, "1", "0"),
        comp("cs", "controlled_current_source", {"gain": 0.2}, "1", "0"),
    ], ["v:1", "s:s", "s:g", "s:i1", "s:out"], 1e-4, 0.02, control=[
        {"id": "s", "kind": "sum", "params": {}, "inputs": ["v1m", "g"]},
        {"id": "g", "kind": "gain", "params": {"k": 0.4}, "inputs": ["s"]},
        {"id": "i1", "kind": "integrator", "params": {}, "inputs": ["mix"]},
        {"id": "mix", "kind": "sum", "params": {}, "inputs": ["gi", "-g"]},
        {"id": "gi", "kind": "gain", "params": {"k": -0.3}, "inputs": ["i1"]},
        {"id": "out", "kind": "limiter", "params": {"min": -2.0, "max": 2.0}, "inputs": ["i1"]},
        {"id": "pi", "kind": "pi_controller", "params": {"kp": 0.5, "ki": 3.0}, "inputs": ["out"]},
        {"id": "cmp", "kind": "comparator", "params": {}, "inputs": ["pi", "v1m"]},
        {"id": "hold", "kind": "delay", "params": {}, "inputs": ["cmp"]},
    ], couplings=[
        {"direction": "meter", "electrical_ref": "1", "signal_ref": "v1m"},
        {"direction": "actuator", "electrical_ref": "cs", "signal_ref": "out"},
    ])


def control_only():
    """No electrical nodes (test_exec.cpp:224-241)."""
    return _doc([], [], ["s:lag", "s:track"], 1e-3, 0.05, control=[
        {"id": "one", "kind": "constant", "params": {"value": 1.0}, "inputs": []},
        {"id": "lag", "kind": "first_order_lag", "params": {"T": 0.01}, "inputs": ["one"]},
        {"id": "track", "kind": "integrator", "params": {}, "inputs": ["lag"]},
    ])


def diverging():
    """Positive actuator feedback diverges -> NonFiniteState (test_exec.cpp:112-139)."""
    return _doc(["1"], [
        comp("r1", "resistor", {"resistance": 1000.0}, "1", "0"),
        comp("cs", "controlled_current_source", {"gain": 1.0}, "1", "0"),
    ], ["v:1"], 1e-3, 1.0, control=[
        {"id": "m2", "kind": "gain", "params": {"k": 4.0}, "inputs": ["v1"]},
        {"id": "b1", "kind": "sum", "params": {}, "inputs": ["m2", "one"]},
        {"id": "one", "kind": "constant", "params": {"value": 1.0}, "inputs": []},
    ], couplings=[
        {"direction": "meter", "electrical_ref": "1", "signal_ref": "v1"},
        {"direction": "actuator", "electrical_ref": "cs", "signal_ref": "b1"},
    ])


def singular_islands():
    """Two ungrounded inductor islands -> SingularMatrix (proj/tests/test_grid.cpp:27-38)."""
    return _doc(["1", "2", "3", "4"], [
        comp("la", "inductor", {"inductance": 1e-3}, "1", "2"),
        comp("lb", "inductor", {"inductance": 2e-3}, "3", "4"),
    ], ["v:1"], 1e-4, 1e-3)


def random_rlc(seed: int, nodes: int = 20, dt: float = 1e-5, duration: float = 0.01):
    """Seeded connected random RLC network (shape of oracles.hpp:187-240; numpy RNG)."""
    rng = np.random.default_rng(seed)
    comps = []

    def add(kind, param, value, a, b):
        comps.append(comp(f"b{100 + len(comps)}", kind, {param: float(value)}, a, b))

    add("resistor", "resistance", rng.uniform(0.5, 2.0), "1", "0")
    for n in range(2, nodes + 1):
        add("resistor", "resistance", rng.uniform(0.5, 2.0), str(int(rng.integers(1, n))), str(n))
    for _ in range(nodes):
        a = int(rng.integers(1, nodes + 1))
        b = int(rng.integers(1, nodes + 1))
        nb = "0" if a == b else str(b)
        k = int(rng.integers(0, 3))
        if k == 0:
            add("resistor", "resistance", rng.uniform(0.5, 2.0), str(a), nb)
        elif k == 1:
            add("inductor", "inductance", 1e-3 * rng.uniform(0.5, 2.0), str(a), nb)
        else:
            add("capacitor", "capacitance", 1e-6 * rng.uniform(0.5, 2.0), str(a), nb)
    comps.append(comp("src", "current_source", {"magnitude": float(rng.uniform(0.5, 2.0)), "frequency": 60.0,
                                                "phase": 0.3}, "1", "0"))
    return _doc([str(n) for n in range(1, nodes + 1)], comps, ["v:1", f"v:{nodes}"], dt, duration)


def subnormal_decay(dt=1e-4, duration=0.6):
    """RC ladder whose node voltages decay through the subnormal range to zero
    (trapezoidal factors down to -1/3 per step): drives the backward sweep's
    division x / u_ii with subnormal and zero x, where a reciprocal-multiply
    division is no longer correctly rounded."""
    return _doc(["1", "2", "3"], [
        comp("c1", "capacitor", {"capacitance": 1e-4, "v0": 1.0}, "1", "0"),
        comp("c2", "capacitor", {"capacitance": 5e-5, "v0": -0.5}, "2", "0"),
        comp("c3", "capacitor", {"capacitance": 2e-4, "v0": 0.25}, "3", "0"),
        comp("r1", "resistor", {"resistance": 1.0}, "1", "0"),
        comp("r12", "resistor", {"resistance": 2.0}, "1", "2"),
        comp("r23", "resistor", {"resistance": 0.5}, "2", "3"),
        comp("r3", "resistor", {"resistance": 0.2}, "3", "0"),
    ], ["v:1", "v:2", "v:3"], dt, duration)


def fuzz(seed: int):
    """Seeded random document exercising every electrical kind, switches with several
    toggles, AC/DC sources and a random control chain fed by meters and driving an
    actuator: the property-style parity set (tests/golden/fuzz/, tools/make_fuzz_fixtures.py)."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(4, 24))
    nodes = [str(k) for k in range(1, n + 1)]
    comps = []
    u = lambda lo, hi: float(rng.uniform(lo, hi))

    def add(kind, params, a, b):
        comps.append(comp(f"c{len(comps):03d}", kind, params, a, b))

    add("resistor", {"resistance": u(0.5, 5.0)}, "1", "0")  # ground path
    for k in range(2, n + 1):  # spanning tree of mixed branches
        a = str(int(rng.integers(1, k)))
        kind = int(rng.integers(0, 4))
        if kind == 0:
            add("resistor", {"resistance": u(0.2, 5.0)}, a, str(k))
        elif kind == 1:
            add("series_rl", {"resistance": u(0.05, 1.0), "inductance": 1e-3 * u(0.2, 3.0)}, a, str(k))
        elif kind == 2:
            add("inductor", {"inductance": 1e-3 * u(0.2, 3.0)}, a, str(k))
        else:
            add("resistor", {"resistance": u(0.2, 5.0)}, a, str(k))
        if rng.random() < 0.5:  # shunt to ground
            if rng.random() < 0.5:
                add("capacitor", {"capacitance": 1e-5 * u(0.3, 3.0)}, str(k), "0")
            else:
                add("resistor", {"resistance": u(5.0, 50.0)}, str(k), "0")
    for _ in range(int(rng.integers(0, 6))):  # meshing branches
        a, b = (str(int(x)) for x in rng.integers(1, n + 1, size=2))
        if a != b:
            add("resistor", {"resistance": u(0.5, 10.0)}, a, b)
    for _ in range(int(rng.integers(1, 4))):  # breakers, possibly several toggles
        a, b = (str(int(x)) for x in rng.integers(1, n + 1, size=2))
        if a == b:
            b = "0"
        times = sorted(float(t) for t in rng.uniform(1e-4, 4e-3, size=int(rng.integers(1, 4))))
        add("switch", {"state": "closed" if rng.random() < 0.5 else "open", "toggle_times": times}, a, b)
    for _ in range(int(rng.integers(1, 3))):  # sources: AC or DC
        a = str(int(rng.integers(1, n + 1)))
        f = 0.0 if rng.random() < 0.3 else u(40.0, 400.0)
        if rng.random() < 0.5:
            add("voltage_source", {"magnitude": u(1.0, 100.0), "frequency": f, "phase": u(-3.0, 3.0),
                                   "rs": u(0.05, 1.0)}, a, "0")
        else:
            add("current_source", {"magnitude": u(0.1, 5.0), "frequency": f, "phase": u(-3.0, 3.0)}, a, "0")
    meter_node = str(int(rng.integers(1, n + 1)))
    act = str(int(rng.integers(1, n + 1)))
    comps.append(comp("act", "controlled_current_source", {"gain": u(-0.05, 0.05)}, act, "0"))
    control = [
        {"id": "k1", "kind": "gain", "params": {"k": u(-0.5, 0.5)}, "inputs": ["vm"]},
        {"id": "lag", "kind": "first_order_lag", "params": {"T": u(1e-4, 1e-2)}, "inputs": ["k1"]},
        {"id": "itg", "kind": "integrator", "params": {}, "inputs": ["lag"]},
        {"id": "pi", "kind": "pi_controller", "params": {"kp": u(0.0, 0.5), "ki": u(0.0, 5.0)}, "inputs": ["lag"]},
        {"id": "sum", "kind": "sum", "params": {}, "inputs": ["pi", "-itg", "one"]},
        {"id": "one", "kind": "constant", "params": {"value": u(-1.0, 1.0)}, "inputs": []},
        {"id": "lim", "kind": "limiter", "params": {"min": -u(0.5, 5.0), "max": u(0.5, 5.0)}, "inputs": ["sum"]},
        {"id": "cmp", "kind": "comparator", "params": {}, "inputs": ["lim", "k1"]},
        {"id": "dly", "kind": "delay", "params": {}, "inputs": ["cmp"]},
    ]
    couplings = [{"direction": "meter", "electrical_ref": meter_node, "signal_ref": "vm"},
                 {"direction": "actuator", "electrical_ref": "act", "signal_ref": "lim"}]
    sw = [c["id"] for c in comps if c["kind"] == "switch"]
    channels = [f"v:{nodes[0]}", f"v:{nodes[-1]}", f"i:{sw[0]}", "s:lim", "s:dly"]
    return _doc(nodes, comps, channels, 1e-5, float(rng.choice([2e-3, 5e-3])), control=control, couplings=couplings)
