"""Bergeron transmission lines and line-split systems (BASELINE C4).

EXTENSION — the reference has no line model (component kinds
proj/include/emtgrid/common.hpp:61-71; "line models are a non-goal",
SPEC.md:227), so nothing here is pinned by the reference; the semantics are
fixed by oracle/emt_oracle.c (case K_BERG) and checked analytically in
tests/test_bergeron.py (open-end voltage doubling, matched-load absorption).

How a line enters the reference's pipeline unchanged: each line END is written
in the reference's own document schema as two placeholder components at the
end's bus — a ``resistor`` of the surge impedance Zc (stamped into G by the
reference compiler like any resistor) and a zero ``current_source`` (the
history-current injection). The reference compiles that document; then
``bergeron_batch`` rewrites each placeholder current source's process record
(schedule text, proj/docs/schedule_format.md) into a NortonBergeron process
(code 20) with a history ring in new arena slots and its line constants in new
const rows. Everything else in the schedule is the reference's output.

Because a Bergeron line adds NO off-diagonal term to G, the two ends of a line
live in decoupled nodal systems: a large network split at its lines is a batch
of small systems ("lanes") whose only coupling is each end reading its peer
end's ring >= K passes late (tau = (K + f) dt, K >= 2). That is how BASELINE C4
(IEEE-39 replicated ~120x, copies coupled by lines) runs: one lane per copy,
peers given per lane in the const table, and on several GPUs one lane shard
per rank exchanging ring rows every K-1 passes (``paper_1903_01081_b200.sharding``).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import schedule as sch

BERGERON_CODE = 20   # kNortonBergeron (csrc/host_schedule.hpp), K_BERG (oracle/emt_oracle.c)
ISRC_CODE = 5        # NortonCurrentSource (proj/include/emtgrid/kernels.hpp:36-59)
NPAR = 7             # [2/Zc, 1-f, f, K, peer_lane, peer_ring_slot, L]


def end_ids(end: str) -> Tuple[str, str]:
    """Placeholder component ids of a line end: (history current source, surge resistor)."""
    return f"{end}_h", f"{end}_z"


def add_line_end(doc: dict, end: str, bus: str, zc: float) -> None:
    """Appends the two placeholder components of one line end at `bus` to a document dict."""
    h, z = end_ids(end)
    doc["components"].append({"id": z, "kind": "resistor", "params": {"resistance": zc}, "terminals": [bus, "0"]})
    doc["components"].append({"id": h, "kind": "current_source",
                              "params": {"magnitude": 0.0, "frequency": 0.0, "phase": 0.0},
                              "terminals": [bus, "0"]})


def delay_split(tau: float, dt: float) -> Tuple[int, float]:
    """tau = (K + f) dt with integer K, 0 <= f < 1 (history read between passes p+1-K and p-K)."""
    r = tau / dt
    k = int(math.floor(r + 1e-9))
    f = r - k
    if abs(f) < 1e-9:
        f = 0.0
    return k, f


@dataclass
class LineSpec:
    """One line end per entry: `ends[e]` = end name, `zc[e]`, `tau[e]`; `peers[l, e]` =
    (peer lane, peer end index) for lane l."""
    ends: List[str]
    zc: List[float]
    tau: List[float]
    peers: np.ndarray  # W x E x 2 ints


def check_symmetric(spec: LineSpec) -> None:
    W, E, _ = spec.peers.shape
    for l in range(W):
        for e in range(E):
            pl, pe = (int(x) for x in spec.peers[l, e])
            if not (0 <= pl < W and 0 <= pe < E):
                raise ValueError(f"lane {l} end {e}: peer ({pl}, {pe}) out of range")
            if tuple(int(x) for x in spec.peers[pl, pe]) != (l, e):
                raise ValueError(f"lane {l} end {e}: peer ({pl}, {pe}) does not point back")
            if spec.zc[e] != spec.zc[pe] or spec.tau[e] != spec.tau[pe]:
                raise ValueError(f"end {e} and its peer end {pe} differ in Zc or tau")


def bergeron_batch(base_schedule: str, base_initial: np.ndarray, component_ids: Sequence[str], spec: LineSpec,
                   const_table: np.ndarray = None) -> sch.Batch:
    """Width-1 reference schedule with line-end placeholders -> W-lane batch whose
    placeholder current sources are NortonBergeron ends coupled as `spec.peers` says.

    `const_table` (consts x W) optionally carries other lane-varying constants
    (e.g. per-copy source phases); the line constants are appended after it."""
    check_symmetric(spec)
    info = sch.parse_info(base_schedule)
    if info.width != 1:
        raise ValueError("bergeron_batch expects a width-1 base schedule")
    W, E, _ = spec.peers.shape
    order = {cid: i for i, cid in enumerate(sorted(component_ids))}
    by_id = {p.id: p for p in info.procs}
    c0, x0 = info.consts, info.extent
    ring_base, par_base, rec = [], [], {}
    nxt = x0
    for e, end in enumerate(spec.ends):
        pid = order[end_ids(end)[0]]
        p = by_id.get(pid)
        if p is None or p.code != ISRC_CODE:
            raise ValueError(f"line end {end}: process {pid} is not the placeholder current source")
        K, f = delay_split(spec.tau[e], info.dt)
        if K < 2:
            raise ValueError(f"line end {end}: travel time {spec.tau[e]} < 2 dt")
        L = 2 * K + 1
        ring_base.append(nxt)
        par_base.append(c0 + NPAR * e)
        rec[pid] = (e, K, f, L)
        nxt += L
    extent = nxt
    consts = c0 + NPAR * E
    ct = np.zeros((consts, W))
    ct[:c0] = info.const_table[:, :1] if const_table is None else const_table
    for e in range(E):
        K, f, L = next((k, ff, ll) for (ee, k, ff, ll) in rec.values() if ee == e)
        b = par_base[e]
        ct[b + 0] = 2.0 / spec.zc[e]
        ct[b + 1] = 1.0 - f
        ct[b + 2] = f
        ct[b + 3] = K
        ct[b + 4] = spec.peers[:, e, 0]
        ct[b + 5] = [ring_base[int(pe)] for pe in spec.peers[:, e, 1]]
        ct[b + 6] = L
    out = []
    for i, ln in enumerate(base_schedule.splitlines()):
        if i == 1:
            f = ln.split()
            f[6] = f"extent={extent}"
            f[7] = f"consts={consts}"
            out.append(" ".join(f))
            continue
        if ln.startswith("P "):
            f = ln.split()
            pid = int(f[1])
            if pid in rec:
                e, K, _, L = rec[pid]
                f[3] = str(BERGERON_CODE)
                f[8] = str(ring_base[e])
                f[9] = str(L)
                f[10] = str(par_base[e])
                f[11] = str(NPAR)
                ln = " ".join(f)
        out.append(ln)
        if ln.startswith(f"CONST {c0 - 1} ") or (c0 == 0 and i == 1):
            for k in range(c0, consts):
                out.append(f"CONST {k} {float(ct[k, 0])!r}")
    text = "\n".join(out) + "\n"
    init = np.zeros((extent, W))
    init[:x0] = sch.replicate_lanes(base_initial, x0, 1, 0, W)
    return sch.Batch(text, ct, init.reshape(-1), W)


# ---------------------------------------------------------------- C4 case

C4_PORTS = [("pa", "b16"), ("pb", "b03"), ("pc", "b26")]  # ring-previous, ring-next, chord


def c4_spec(copies: int, zc: float = 300.0, tau: float = 0.33e-3) -> LineSpec:
    """Copies coupled by lines: ring (port a of copy r <-> port b of copy r-1) and
    chords (port c of copy r <-> port c of copy r + R/2)."""
    if copies < 2 or copies % 2:
        raise ValueError("C4 needs an even number (>= 2) of copies")
    peers = np.zeros((copies, 3, 2), dtype=np.int64)
    for r in range(copies):
        peers[r, 0] = ((r - 1) % copies, 1)
        peers[r, 1] = ((r + 1) % copies, 0)
        peers[r, 2] = ((r + copies // 2) % copies, 2)
    return LineSpec([p for p, _ in C4_PORTS], [zc] * 3, [tau] * 3, peers)


def c4_document(duration: float = 1.0, dt: float = 50e-6, zc: float = 300.0) -> str:
    """One IEEE-39 copy with the three C4 line-end placeholders (reference JSON schema)."""
    from . import cases
    doc = json.loads(cases.ieee39_document(duration=duration, dt=dt,
                                           channels=["v:b16", "v:b03", "v:b26", "i:pa_h", "i:pc_h"]))
    for end, bus in C4_PORTS:
        add_line_end(doc, end, bus, zc)
    return json.dumps(doc, indent=1) + "\n"


def generator_phase_slots(info: sch.ScheduleInfo) -> List[int]:
    """Const slots of every voltage source's phase (CompanionSpec [1/rs, mag, omega, phase],
    proj/include/emtgrid/kernels.hpp:92-105)."""
    return [p.par + 3 for p in info.procs if p.code == 4 and p.par_len >= 4]


def c4_batch(base_schedule: str, base_initial: np.ndarray, component_ids: Sequence[str], copies: int,
             zc: float = 300.0, tau: float = 0.33e-3, swing: float = 0.2) -> sch.Batch:
    """C4: `copies` IEEE-39 copies as lanes, each copy's generator angles shifted by
    swing*sin(2 pi r / R) rad so power flows through the coupling lines."""
    info = sch.parse_info(base_schedule)
    ct = np.repeat(info.const_table[:, :1], copies, axis=1)
    shift = swing * np.sin(2.0 * np.pi * np.arange(copies) / copies)
    for k in generator_phase_slots(info):
        ct[k] = ct[k] + shift
    return bergeron_batch(base_schedule, base_initial, component_ids, c4_spec(copies, zc, tau), ct)


def single_line_document(e_volts: float = 1000.0, zc: float = 400.0, rs: float = 400.0, load: float = 0.0,
                         dt: float = 50e-6, duration: float = 0.02) -> str:
    """Analytic test case: DC source (rs) -> bus `a` -- line -- bus `b` (open, or a
    resistive `load` to ground when load > 0). Ends: "la" at a, "lb" at b."""
    doc = {
        "nodes": ["a", "b"],
        "components": [
            {"id": "src", "kind": "voltage_source",
             "params": {"magnitude": e_volts, "frequency": 0.0, "phase": 0.0, "rs": rs}, "terminals": ["a", "0"]},
        ],
        "control": [], "couplings": [],
        "task": {"dt": dt, "duration": duration, "channels": ["v:a", "v:b"], "device_profile": "cpu-serial",
                 "strategy": "serial"},
    }
    if load > 0.0:
        doc["components"].append({"id": "rl", "kind": "resistor", "params": {"resistance": load},
                                  "terminals": ["b", "0"]})
    add_line_end(doc, "la", "a", zc)
    add_line_end(doc, "lb", "b", zc)
    return json.dumps(doc, indent=1) + "\n"


def single_line_spec(zc: float, tau: float, width: int = 1) -> LineSpec:
    peers = np.zeros((width, 2, 2), dtype=np.int64)
    for l in range(width):
        peers[l, 0] = (l, 1)
        peers[l, 1] = (l, 0)
    return LineSpec(["la", "lb"], [zc, zc], [tau, tau], peers)


# ---------------------------------------------------------------- document kind

LINE_KIND = "transmission_line"
LINE_PARAMS = ("surge_impedance", "travel_time")


class LineDocumentError(ValueError):
    """A `transmission_line` component failed validation; `code` names the reference's
    ErrorCode (proj/include/emtgrid/common.hpp:11-33) the check mirrors, `where` its id."""

    def __init__(self, code: str, where: str, message: str):
        super().__init__(f"{code}: {message} (at {where})")
        self.code, self.where = code, where


def line_end_names(line_id: str) -> Tuple[str, str]:
    """The two ends of line `line_id` (placeholder pairs `<end>_h` / `<end>_z`)."""
    return f"{line_id}__a", f"{line_id}__b"


def expand_document(document: str) -> Tuple[str, LineSpec]:
    """The `transmission_line` document kind (EXTENSION): parse and
    validate every line the way the reference's check_component validates its kinds
    (proj/src/model.cpp:154-222: arity, allowed parameter keys, strictly positive
    finite values; identifiers and node references as in parse, model.cpp), then
    stamp each line as its two placeholder ends (add_line_end: surge resistor +
    history current source at each terminal bus). Returns the reference-schema
    document (compile it with the reference's parse_model -> compile_task) and the
    width-1 LineSpec pairing each line's two ends, for `bergeron_batch`.

        {"id": "L1", "kind": "transmission_line", "terminals": ["b16", "b03"],
         "params": {"surge_impedance": 300.0, "travel_time": 3.3e-4}}

    A line's ends are Norton equivalents to ground at its two buses (lossless
    Bergeron model); it adds no off-diagonal term to G, so the buses it joins may
    lie in otherwise separate subnetworks (each needs its own ground path)."""
    doc = json.loads(document)
    comps = doc.get("components", [])
    nodes = set(doc.get("nodes", []))
    dt = float(doc.get("task", {}).get("dt", 0.0))
    ids = [c.get("id", "") for c in comps]
    out = dict(doc)
    out["components"] = []
    ends, zcs, taus = [], [], []
    for c in comps:
        if c.get("kind") != LINE_KIND:
            out["components"].append(c)
            continue
        where = c.get("id", "")
        if not where:
            raise LineDocumentError("MalformedDocument", "components", "transmission line without an id")
        if ids.count(where) > 1:
            raise LineDocumentError("DuplicateIdentifier", where, "component id declared twice")
        terms = c.get("terminals", [])
        if len(terms) != 2:
            raise LineDocumentError("InvalidParameter", where,
                                    f"transmission_line needs 2 terminals, got {len(terms)}")
        for t in terms:
            if t == "0":
                raise LineDocumentError("InvalidParameter", where, "a line end must sit at a bus, not ground")
            if t not in nodes:
                raise LineDocumentError("DanglingReference", t, f"terminal of {where} is not a declared node")
        if terms[0] == terms[1]:
            raise LineDocumentError("InvalidParameter", where, "line ends must be two different buses")
        params = c.get("params", {})
        for k in params:
            if k not in LINE_PARAMS:
                raise LineDocumentError("InvalidParameter", where, f"unknown parameter '{k}'")
        vals = []
        for k in LINE_PARAMS:
            v = params.get(k)
            if not isinstance(v, (int, float)) or isinstance(v, bool):
                raise LineDocumentError("InvalidParameter", where, f"missing numeric parameter '{k}'")
            v = float(v)
            if not (v > 0.0) or not math.isfinite(v):
                raise LineDocumentError("InvalidParameter", where, f"{k} must be strictly positive")
            vals.append(v)
        zc, tau = vals
        if dt > 0.0 and delay_split(tau, dt)[0] < 2:
            raise LineDocumentError("InvalidParameter", where, "travel_time must be at least 2 dt")
        for end, bus in zip(line_end_names(where), terms):
            for pid in end_ids(end):
                if pid in ids:
                    raise LineDocumentError("DuplicateIdentifier", pid, "collides with a line-end placeholder id")
            add_line_end(out, end, bus, zc)
            ends.append(end)
            zcs.append(zc)
            taus.append(tau)
    E = len(ends)
    peers = np.zeros((1, E, 2), dtype=np.int64)
    for e in range(0, E, 2):  # the two ends of one line point at each other
        peers[0, e] = (0, e + 1)
        peers[0, e + 1] = (0, e)
    return json.dumps(out, indent=1) + "\n", LineSpec(ends, zcs, taus, peers)


def document_batch(document: str, compile_fn) -> sch.Batch:
    """A document with `transmission_line` components -> executable width-1 batch:
    expand_document, then `compile_fn(reference_document) -> (schedule text, initial
    arena)` (the reference compiler, parse_model -> compile_task), then the line ends
    become NortonBergeron processes (bergeron_batch)."""
    expanded, spec = expand_document(document)
    schedule, initial = compile_fn(expanded)
    cids = [c["id"] for c in json.loads(expanded)["components"]]
    if not spec.ends:
        info = sch.parse_info(schedule)
        return sch.Batch(schedule, info.const_table, np.asarray(initial, dtype=np.float64), 1)
    return bergeron_batch(schedule, np.asarray(initial, dtype=np.float64), cids, spec)
