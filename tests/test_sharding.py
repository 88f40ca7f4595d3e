"""Multi-GPU host logic on CPU: lane shards, max-over-ranks timing, final gather (gloo, world 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_01081_b200 import cases, sharding


def test_shard_bounds_cover_exactly():
    for W in (1, 7, 1000, 1012):
        for world in (1, 2, 3, 8):
            if world > W:
                continue
            spans = [sharding.shard_bounds(W, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == W
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_n1_sweep_matches_baseline_grid_at_n1():
    base = cases.n1_scenarios(1000)
    sweep = sharding.n1_sweep(1000)
    assert [(b, t) for b, t in base] == sweep
    big = sharding.n1_sweep(8000)
    assert len(set(big)) == 8000  # weak-scaling sweeps stay distinct


def test_factor_count_union():
    assert sharding.combine_factor_counts([[0, 2000, 2200], [0, 2200, 6000]]) == 4


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = sharding.shard_bounds(10, world, rank)
    local = np.arange(lo, hi, dtype=np.float64)
    t = sharding.reduce_max(dist, float(rank + 1) * 1.5)
    g = sharding.gather_digests(dist, sharding.digest(local), world)
    out[rank] = (t, g.tolist())
    dist.destroy_process_group()


def test_gloo_world2_reduce_and_gather():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for rank in (0, 1):
        t, g = out[rank]
        assert t == 3.0  # max over ranks
        g = np.array(g)
        assert np.allclose(g[0], sharding.digest(np.arange(0, 5.0)))
        assert np.allclose(g[1], sharding.digest(np.arange(5, 10.0)))


def _ring_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, cols = 10, 7
    lo, hi = sharding.shard_bounds(W, world, rank)
    mirror = torch.full((W, cols), -1.0, dtype=torch.float64)
    mirror[lo:hi] = torch.arange(lo * cols, hi * cols, dtype=torch.float64).reshape(hi - lo, cols)
    sharding.exchange_rings(dist, mirror, lo, hi)
    out[rank] = mirror.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_exchange_gloo(world):
    """Line-split boundary exchange: after one exchange every rank holds every lane's rows."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(_ring_worker, args=(world, port, out), nprocs=world, join=True)
    want = np.arange(10 * 7, dtype=np.float64).reshape(10, 7)
    for r in range(world):
        assert np.array_equal(out[r], want)
