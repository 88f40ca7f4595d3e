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
