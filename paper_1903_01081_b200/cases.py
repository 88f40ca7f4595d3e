"""Synthetic case documents in the reference's JSON model format.

The reference bundles only proj/data/feeder33_pv3.json; BASELINE.json's
configs C2/C3 name an IEEE 39-bus case, which is generated here in the
reference's document schema (parse_model, /root/reference/proj/src/model.cpp:476-590;
component kinds proj/include/emtgrid/common.hpp:61-71).

IEEE-39 data: branch list and per-unit R/X/B are the New England 39-bus
system (MATPOWER case39, 100 MVA base, 345 kV) as entered offline from
memory; load P/Q and generator voltage/angle are the case's power-flow
values, rounded. It is labelled ``ieee39-synthetic`` because it was not
checked against an official data file. EMT modelling choices (single-phase
equivalent, 60 Hz):
  * generator g at bus k: ``voltage_source`` bus→ground, peak
    Vm·345 kV·sqrt(2/3), phase = power-flow angle, rs = 0.5 Ω;
  * each of the 46 branches: ``switch`` (closed, toggle_times=[never])
    from bus i to a mid node, then ``series_rl`` mid→bus j (transformers
    get R = 0.002·X when the case has R = 0);
  * the 19 loads: ``series_rl`` bus→ground from P, Q at 345 kV;
  * line charging: one ``capacitor`` per bus holding half of every
    incident line's B.
Node order = matrix order (the reference factorizes with the identity
permutation, proj/src/sparse.cpp:44-77): mid nodes first, buses in a
greedy minimum-degree order, which keeps LU fill and the triangular-solve
depth small while staying bit-compatible with the reference.
"""
from __future__ import annotations

import json
import math

NEVER = 1.0e9  # sentinel toggle time: never reached inside any run

# (from, to, r_pu, x_pu, b_pu, is_transformer)
IEEE39_BRANCHES = [
    (1, 2, 0.0035, 0.0411, 0.6987, 0), (1, 39, 0.0010, 0.0250, 0.7500, 0),
    (2, 3, 0.0013, 0.0151, 0.2572, 0), (2, 25, 0.0070, 0.0086, 0.1460, 0),
    (2, 30, 0.0000, 0.0181, 0.0000, 1), (3, 4, 0.0013, 0.0213, 0.2214, 0),
    (3, 18, 0.0011, 0.0133, 0.2138, 0), (4, 5, 0.0008, 0.0128, 0.1342, 0),
    (4, 14, 0.0008, 0.0129, 0.1382, 0), (5, 6, 0.0002, 0.0026, 0.0434, 0),
    (5, 8, 0.0008, 0.0112, 0.1476, 0), (6, 7, 0.0006, 0.0092, 0.1130, 0),
    (6, 11, 0.0007, 0.0082, 0.1389, 0), (6, 31, 0.0000, 0.0250, 0.0000, 1),
    (7, 8, 0.0004, 0.0046, 0.0780, 0), (8, 9, 0.0023, 0.0363, 0.3804, 0),
    (9, 39, 0.0010, 0.0250, 1.2000, 0), (10, 11, 0.0004, 0.0043, 0.0729, 0),
    (10, 13, 0.0004, 0.0043, 0.0729, 0), (10, 32, 0.0000, 0.0200, 0.0000, 1),
    (12, 11, 0.0016, 0.0435, 0.0000, 1), (12, 13, 0.0016, 0.0435, 0.0000, 1),
    (13, 14, 0.0009, 0.0101, 0.1723, 0), (14, 15, 0.0018, 0.0217, 0.3660, 0),
    (15, 16, 0.0009, 0.0094, 0.1710, 0), (16, 17, 0.0007, 0.0089, 0.1342, 0),
    (16, 19, 0.0016, 0.0195, 0.3040, 0), (16, 21, 0.0008, 0.0135, 0.2548, 0),
    (16, 24, 0.0003, 0.0059, 0.0680, 0), (17, 18, 0.0007, 0.0082, 0.1319, 0),
    (17, 27, 0.0013, 0.0173, 0.3216, 0), (19, 20, 0.0007, 0.0138, 0.0000, 1),
    (19, 33, 0.0007, 0.0142, 0.0000, 1), (20, 34, 0.0009, 0.0180, 0.0000, 1),
    (21, 22, 0.0008, 0.0140, 0.2565, 0), (22, 23, 0.0006, 0.0096, 0.1846, 0),
    (22, 35, 0.0000, 0.0143, 0.0000, 1), (23, 24, 0.0022, 0.0350, 0.3610, 0),
    (23, 36, 0.0005, 0.0272, 0.0000, 1), (25, 26, 0.0032, 0.0323, 0.5310, 0),
    (25, 37, 0.0006, 0.0232, 0.0000, 1), (26, 27, 0.0014, 0.0147, 0.2396, 0),
    (26, 28, 0.0043, 0.0474, 0.7802, 0), (26, 29, 0.0057, 0.0625, 1.0290, 0),
    (28, 29, 0.0014, 0.0151, 0.2490, 0), (29, 38, 0.0008, 0.0156, 0.0000, 1),
]
# bus: (P MW, Q MVAr)
IEEE39_LOADS = {
    3: (322.0, 2.4), 4: (500.0, 184.0), 7: (233.8, 84.0), 8: (522.0, 176.0), 12: (7.5, 88.0),
    15: (320.0, 153.0), 16: (329.0, 32.3), 18: (158.0, 30.0), 20: (628.0, 103.0), 21: (274.0, 115.0),
    23: (247.5, 84.6), 24: (308.6, -92.2), 25: (224.0, 47.2), 26: (139.0, 17.0), 27: (281.0, 75.5),
    28: (206.0, 27.6), 29: (283.5, 26.9), 31: (9.2, 4.6), 39: (1104.0, 250.0),
}
# bus: (Vm pu, angle deg)
IEEE39_GENS = {
    30: (1.0475, -3.65), 31: (0.9820, 0.00), 32: (0.9831, 2.57), 33: (0.9972, 4.42), 34: (1.0123, 3.37),
    35: (1.0493, 5.65), 36: (1.0635, 8.35), 37: (1.0278, 2.43), 38: (1.0265, 7.81), 39: (1.0300, -10.05),
}

V_BASE = 345.0e3
S_BASE = 100.0e6
FREQ = 60.0


def _bus(k: int) -> str:
    return f"b{k:02d}"


def _min_degree_order(nodes, edges):
    """Greedy minimum-degree elimination order (ties: name)."""
    adj = {n: set() for n in nodes}
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    order = []
    remaining = set(nodes)
    while remaining:
        v = min(remaining, key=lambda n: (len(adj[n] & remaining), n))
        nbrs = adj[v] & remaining
        for a in nbrs:
            adj[a] |= nbrs - {a}
        remaining.remove(v)
        order.append(v)
    return order


def ieee39_document(duration: float = 1.0, dt: float = 50e-6, channels=None, outage: int = -1,
                    fault_time: float = NEVER) -> str:
    """IEEE-39 EMT document; ``outage`` = branch index whose breaker opens at ``fault_time``."""
    zb = V_BASE ** 2 / S_BASE
    w = 2.0 * math.pi * FREQ
    comps = []
    shunt_b = {k: 0.0 for k in range(1, 40)}
    bus_edges = []
    mids = []
    for idx, (i, j, r, x, b, xf) in enumerate(IEEE39_BRANCHES):
        mid = f"m{idx:02d}"
        mids.append(mid)
        r_ohm = (r if r > 0 else 0.002 * x) * zb
        l_h = x * zb / w
        toggle = [fault_time] if idx == outage else [NEVER]
        comps.append({"id": f"sw{idx:02d}", "kind": "switch", "params": {"state": "closed", "toggle_times": toggle},
                      "terminals": [_bus(i), mid]})
        comps.append({"id": f"ln{idx:02d}", "kind": "series_rl",
                      "params": {"resistance": r_ohm, "inductance": l_h}, "terminals": [mid, _bus(j)]})
        shunt_b[i] += b / 2.0
        shunt_b[j] += b / 2.0
        bus_edges.append((_bus(i), _bus(j)))
    for k, (p_mw, q_mvar) in sorted(IEEE39_LOADS.items()):
        p = p_mw * 1e6
        q = max(q_mvar, 0.2 * p_mw) * 1e6
        den = p * p + q * q
        comps.append({"id": f"ld{k:02d}", "kind": "series_rl",
                      "params": {"resistance": V_BASE ** 2 * p / den, "inductance": V_BASE ** 2 * q / den / w},
                      "terminals": [_bus(k), "0"]})
    for k, (vm, ang) in sorted(IEEE39_GENS.items()):
        comps.append({"id": f"gen{k:02d}", "kind": "voltage_source",
                      "params": {"magnitude": vm * V_BASE * math.sqrt(2.0 / 3.0), "frequency": FREQ,
                                 "phase": math.radians(ang), "rs": 0.5},
                      "terminals": [_bus(k), "0"]})
    for k in range(1, 40):
        if shunt_b[k] > 0.0:
            comps.append({"id": f"cb{k:02d}", "kind": "capacitor",
                          "params": {"capacitance": shunt_b[k] / zb / w}, "terminals": [_bus(k), "0"]})
    buses = [_bus(k) for k in range(1, 40)]
    nodes = mids + _min_degree_order(buses, bus_edges)
    if channels is None:
        channels = ["v:b16", "v:b03", "v:b39", "i:ln16", "i:ld39"]
    doc = {
        "nodes": nodes,
        "components": comps,
        "control": [],
        "couplings": [],
        "task": {"dt": dt, "duration": duration, "channels": channels, "device_profile": "cpu-serial",
                 "strategy": "serial"},
    }
    return json.dumps(doc, indent=1) + "\n"


def n1_scenarios(count: int = 1000, n_branches: int = len(IEEE39_BRANCHES), n_times: int = 22):
    """N-1 sweep: lane s -> (branch s // 22, t_f = 0.10 + 0.01*(s % 22)),
    outage-major, truncated to ``count``."""
    out = []
    for s in range(min(count, n_branches * n_times)):
        out.append((s // n_times, 0.10 + 0.01 * (s % n_times)))
    return out
