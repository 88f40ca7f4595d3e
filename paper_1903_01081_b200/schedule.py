"""Host-side helpers over the reference's schedule / state text formats.

Formats: /root/reference/proj/docs/schedule_format.md (`.cgmsched` v1 and
`STATE v1`). Widening a compiled width-1 schedule to W scenario lanes is the
schedule-level form of the reference's `vectorize` (proj/src/cgm.cpp:377-400):
structure is shared, only the slot-major constant table (and initial arena)
gain a lane axis. It also admits array-valued overrides such as an N-1
breaker's `toggle_times`, which `apply_overrides` (proj/src/cgm.cpp:22-48)
cannot express.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np


@dataclass
class ProcRecord:
    id: int
    kind: int
    code: int
    out: int
    out2: int
    state: int
    state_len: int
    par: int
    par_len: int


@dataclass
class ScheduleInfo:
    width: int
    layers: int
    dt: float
    steps: int
    nodes: int
    comps: int
    blocks: int
    extent: int
    consts: int
    const_table: np.ndarray  # consts x width
    procs: List[ProcRecord]
    channels: List[Tuple[str, int]]


def _kv(tok: str) -> str:
    return tok.split("=", 1)[1]


def parse_info(text: str) -> ScheduleInfo:
    lines = text.splitlines()
    h = lines[0].split()
    m = lines[1].split()
    width = int(_kv(h[4]))
    info = ScheduleInfo(width=width, layers=int(_kv(h[3])), dt=float(_kv(m[1])), steps=int(_kv(m[2])),
                        nodes=int(_kv(m[3])), comps=int(_kv(m[4])), blocks=int(_kv(m[5])), extent=int(_kv(m[6])),
                        consts=int(_kv(m[7])), const_table=None, procs=[], channels=[])
    ct = np.zeros((info.consts, width))
    for ln in lines[2:]:
        if ln.startswith("CONST "):
            f = ln.split()
            ct[int(f[1])] = [float(x) for x in f[2:2 + width]]
        elif ln.startswith("P "):
            f = ln.split()
            info.procs.append(ProcRecord(int(f[1]), int(f[2]), int(f[3]), int(f[5]), int(f[7]), int(f[8]), int(f[9]),
                                         int(f[10]), int(f[11])))
        elif ln.startswith("CHANNEL "):
            f = ln.split()
            info.channels.append((f[1], int(f[2])))
    info.const_table = ct
    return info


def parse_state(text: str) -> Tuple[np.ndarray, int]:
    """parse_state (proj/src/schedule.cpp:599-622) -> (flat arena, width)."""
    lines = text.split("\n")
    h = lines[0].split()
    extent, width = int(_kv(h[2])), int(_kv(h[3]))
    body = " ".join(lines[1:1 + extent])
    arena = np.array(body.split(), dtype=np.float64)
    if arena.size != extent * width:
        raise ValueError("truncated state file")
    return arena, width


def format_state(arena: np.ndarray, extent: int, width: int) -> str:
    """serialize_state (proj/src/schedule.cpp:582-597), %.17g round-trip form."""
    a = np.asarray(arena, dtype=np.float64).reshape(extent, width)
    out = [f"STATE v1 extent={extent} width={width}"]
    out += [" ".join("%.17g" % x for x in row) for row in a]
    return "\n".join(out) + "\n"


def widen_text(text: str, const_table: np.ndarray) -> str:
    """Re-serialises a schedule with a new (consts x W) table: header width and CONST rows."""
    consts, width = const_table.shape
    out = []
    for i, ln in enumerate(text.splitlines()):
        if i == 0:
            f = ln.split()
            f[4] = f"width={width}"
            out.append(" ".join(f))
        elif ln.startswith("CONST "):
            k = int(ln.split()[1])
            out.append(f"CONST {k} " + " ".join(repr(float(x)) for x in const_table[k]))
        else:
            out.append(ln)
    return "\n".join(out) + "\n"


def replicate_lanes(arr_slot_major: np.ndarray, rows: int, width_in: int, lane: int, width_out: int) -> np.ndarray:
    """Broadcasts lane `lane` of a slot-major (rows x width_in) array to width_out lanes."""
    a = np.asarray(arr_slot_major, dtype=np.float64).reshape(rows, width_in)[:, lane]
    return np.repeat(a[:, None], width_out, axis=1)


def switch_toggle_slots(info: ScheduleInfo) -> Dict[int, int]:
    """process id (== canonical component index) of each NortonSwitch -> const slot of its
    first toggle time (CompanionSpec layout [g_on, g_off, initial, t0, ...],
    proj/include/emtgrid/kernels.hpp:92-105)."""
    return {p.id: p.par + 3 for p in info.procs if p.code == 7 and p.par_len > 3}


@dataclass
class Batch:
    schedule: str            # width-1 base schedule text
    const_table: np.ndarray  # consts x W
    initial: np.ndarray      # extent x W, flattened slot-major
    width: int

    def text(self) -> str:
        """Full-width schedule text (for consumers that only read text, e.g. the reference)."""
        return widen_text(self.schedule, self.const_table)


def n1_batch(base_schedule: str, base_initial: np.ndarray, component_ids: Sequence[str],
             scenarios: Sequence[Tuple[str, float]]) -> Batch:
    """N-1 batch: lane s opens breaker scenarios[s][0] at time scenarios[s][1].

    `component_ids` are the document's component ids; the canonical order is
    ascending id (canonical_component_order, proj/src/model.cpp:708-716) and the
    Norton process id equals that index (Cgm::norton_id, proj/include/emtgrid/cgm.hpp:66)."""
    info = parse_info(base_schedule)
    order = {cid: i for i, cid in enumerate(sorted(component_ids))}
    slots = switch_toggle_slots(info)
    W = len(scenarios)
    ct = np.repeat(info.const_table[:, :1], W, axis=1)
    for lane, (comp, t_f) in enumerate(scenarios):
        ct[slots[order[comp]], lane] = t_f
    init = replicate_lanes(base_initial, info.extent, info.width, 0, W).reshape(-1)
    return Batch(base_schedule, ct, init, W)


def rows_json(rows) -> str:
    return json.dumps(rows)


def pv_grid(n_irr: int = 64, n_temp: int = 64, irr=(400.0, 1100.0), temp=(5.0, 45.0)) -> List[Tuple[float, float]]:
    """gen_scenarios row order (proj/src/bench.cpp:137-146): irradiance-major, temperature inner."""
    return [(float(i), float(t)) for i in np.linspace(irr[0], irr[1], n_irr) for t in np.linspace(temp[0], temp[1], n_temp)]


def pv_sweep_batch(base_schedule: str, base_initial: np.ndarray, pv_map: dict,
                   scenarios: Sequence[Tuple[float, float]]) -> Batch:
    """Shared-G batch (BASELINE C5): lane s sets every PV's (irradiance, temperature).

    The override only changes the photocurrent J = 10 (irr/1000)(1 + 0.0004 (temp-25))
    (proj/src/model.cpp:306-309) — each PV current source's magnitude constant and
    +-J initial branch currents — so G is identical across lanes. `pv_map` (the case
    data's "pv_sweep" record) names those slots; tools/make_fixtures.py derives it
    from the reference's own vectorize and tests/test_schedule_host.py pins this
    widening against it bit for bit."""
    info = parse_info(base_schedule)
    W = len(scenarios)
    j = np.array([10.0 * (irr / 1000.0) * (1.0 + 0.0004 * (tmp - 25.0)) for irr, tmp in scenarios])
    ct = np.repeat(info.const_table[:, :1], W, axis=1)
    for k in pv_map["const_slots"]:
        ct[k, :] = j
    init = replicate_lanes(base_initial, info.extent, info.width, 0, W).reshape(info.extent, W)
    for k, sign in pv_map["init_slots"]:
        init[k, :] = j if sign > 0 else -j
    return Batch(base_schedule, ct, init.reshape(-1), W)
