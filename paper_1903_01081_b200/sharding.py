"""Multi-GPU scenario sharding.

Scenario lanes are independent units, so an N-GPU sweep is N contiguous lane
shards — one process per GPU, no data-path collective. The only inter-rank
traffic is the run-time reduction (max over ranks of the device time) and a
final result gather (per-rank waveform digests / event counts).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def shard_bounds(width: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous lane range [lo, hi) of `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * width // world, (rank + 1) * width // world


def n1_sweep(total: int, n_branches: int = 46, n_times: int = 22, t0: float = 0.10, dt_f: float = 0.01,
             refine: float = 0.001) -> List[Tuple[int, float]]:
    """Scenario s -> (breaker s // n_times mod n_branches, fault time). The first
    n_branches*n_times scenarios are the BASELINE C3 grid (0.10-0.31 s, outage-major);
    larger sweeps (weak scaling, 1000 scenarios per GPU) repeat the grid with the
    fault times shifted by `refine` seconds per repetition."""
    grid = n_branches * n_times
    out = []
    for s in range(total):
        rep, k = divmod(s, grid)
        out.append(((k // n_times) % n_branches, t0 + dt_f * (k % n_times) + refine * rep))
    return out


def digest(values: np.ndarray) -> np.ndarray:
    """Order-independent per-rank result digest: (sum, sum of squares, max |x|)."""
    v = np.asarray(values, dtype=np.float64)
    return np.array([float(v.sum()), float((v * v).sum()), float(np.abs(v).max() if v.size else 0.0)])


def reduce_max(dist, value: float, device=None) -> float:
    """Max over ranks (timing is reported as the slowest rank)."""
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_digests(dist, local: np.ndarray, world: int, device=None) -> np.ndarray:
    """Final result gather: every rank's digest, rank-ordered."""
    import torch
    t = torch.tensor(local, dtype=torch.float64, device=device)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return np.stack([p.cpu().numpy() for p in parts])


def combine_factor_counts(per_rank_refactor_steps: Sequence[Sequence[int]]) -> int:
    """Global factor_count of a sharded run: the reference counts passes in which ANY
    lane refactorised (proj/src/exec.cpp:177-203), i.e. the union over shards."""
    steps = set()
    for s in per_rank_refactor_steps:
        steps.update(int(x) for x in s)
    return len(steps)


# ---------------------------------------------------------------- line-split systems (C4)

def exchange_rings(dist, mirror, lo: int, hi: int) -> None:
    """Boundary exchange of a line-split system: every rank contributes its lanes'
    rows [lo, hi) of the lane-major line-end history mirror (engine.ring()) and
    receives everyone else's. One collective per launch of <= K-1 passes; the
    Bergeron travel time gives those K-1 passes of slack."""
    import torch
    if mirror.is_cuda and dist.get_backend() == "gloo":  # host-staged (tests: several ranks, one GPU)
        host = mirror.cpu()
        exchange_rings(dist, host, lo, hi)
        mirror.copy_(host)
        return
    world = dist.get_world_size()
    W = mirror.shape[0]
    bounds = [shard_bounds(W, world, r) for r in range(world)]
    width = max(b - a for a, b in bounds)
    send = torch.zeros((width,) + tuple(mirror.shape[1:]), dtype=mirror.dtype, device=mirror.device)
    send[: hi - lo] = mirror[lo:hi]
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send)
    for r, (a, b) in enumerate(bounds):
        if r != dist.get_rank():
            mirror[a:b] = parts[r][: b - a]


class LineSplitShard:
    """One rank's lanes of a line-coupled batch: an Engine over [lo, hi).

    exchange="device" (default with several ranks): rank 0 allocates the
    line-history mirror and a progress word per CTA of the whole system with
    CUDA IPC; every rank's engine attaches both (emt_engine_attach_lines) and
    runs its launches persistently — CTAs write their histories straight into
    the shared mirror over NVLink and wait on the other ranks' progress words,
    with no host involvement. exchange="host": launches of at most
    `max_chunk` (= K-1) passes and a torch.distributed all-gather of the
    mirror rows after each one. With world == 1 it is a plain engine."""

    def __init__(self, dist, batch, lo: int, hi: int, device: int = 0, exchange: str = "", **engine_kw):
        import os
        import torch
        from . import engine
        self.dist, self.lo, self.hi = dist, lo, hi
        self.eng = engine.Engine(batch.schedule, batch.initial, const_table=batch.const_table, width=batch.width,
                                 device=device, lane_begin=lo, lane_count=hi - lo, **engine_kw)
        ptr, lanes, cols, self.max_chunk = self.eng.ring()
        self.world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
        self.exchange = exchange or os.environ.get("EMTB200_LINE_EXCHANGE", "device")
        self.mirror = None
        self._ipc = []
        if not ptr or self.world == 1:
            return
        if self.exchange == "device" and self.eng.kernel == engine.KERNEL_SPECIALISED:
            rank = dist.get_rank()
            # each engine's own CTA count (emt_engine_ctas), gathered: no lanes-per-CTA assumption
            mine = torch.tensor([self.eng.ctas()[0]], dtype=torch.int64)
            if dist.get_backend() == "nccl":
                mine = mine.cuda(device)
            parts = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(parts, mine)
            ctas = [int(p.item()) for p in parts]
            total = sum(ctas)
            offset = sum(ctas[:rank])
            mb, pb = lanes * cols * 8, total * 4
            hbuf = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                mptr, mh = engine.ipc_alloc(device, mb)
                pptr, ph = engine.ipc_alloc(device, pb)
                self._ipc = [("free", mptr), ("free", pptr)]
                hbuf[:64] = torch.frombuffer(bytearray(mh), dtype=torch.uint8)
                hbuf[64:] = torch.frombuffer(bytearray(ph), dtype=torch.uint8)
            if dist.get_backend() == "nccl":
                hb = hbuf.cuda(device)
                dist.broadcast(hb, 0)
                hbuf = hb.cpu()
            else:
                dist.broadcast(hbuf, 0)
            if rank != 0:
                raw = bytes(hbuf.numpy().tobytes())
                mptr = engine.ipc_open(device, raw[:64])
                pptr = engine.ipc_open(device, raw[64:])
                self._ipc = [("close", mptr), ("close", pptr)]
            self.eng.attach_lines(mptr, pptr, offset, total, system_scope=os.environ.get("EMTB200_LINE_SCOPE", "sys") == "sys")
            dist.barrier()  # every rank's rows and progress words initialised before any launch
            self.max_chunk = 0
            return
        # host exchange: peers' rows arrive by all-gather after every launch of K-1 passes
        self.exchange = "host"
        self.mirror = torch.zeros((lanes, cols), dtype=torch.float64, device=torch.device("cuda", device))
        self.eng.attach_ring(self.mirror.data_ptr())

    def advance(self, steps: int) -> None:
        import torch
        if self.world == 1 or self.mirror is None or self.max_chunk <= 0:
            self.eng.advance(steps)
            return
        done = 0
        while done < steps:
            n = min(self.max_chunk, steps - done)
            self.eng.advance(n)
            self.eng.sync()
            exchange_rings(self.dist, self.mirror, self.lo, self.hi)
            torch.cuda.current_stream().synchronize()
            done += n

    def reload(self, initial, const_table=None) -> None:
        """New batch on every rank: reset (own progress words), then a barrier so no
        rank launches against another rank's stale progress."""
        self.eng.load(initial, const_table)
        self.eng.sync()  # the mirror rows and progress resets have landed before peers launch
        if self.world > 1:
            self.dist.barrier()
