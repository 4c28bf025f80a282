"""The multi-GPU sweep logic (sharding, all-gather of traces, argmin tie-break) on CPU with gloo,
world_size 2 and 3, against a fake analytic solver; plus shard properties.  (The CUDA engine is
per-rank and needs no collective; the real NCCL path is the same code in bench.py.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_08201_b200.sweep import Sweep, shard_indices


def fake_tau(v):
    """Analytic stand-in for trace(E X(v)): the 1-DOF closed form 2/c + c/(2 w^2) with c = 0.1 + v0
    (minimum at c = 2w, i.e. v0 = 2w - 0.1), plus a small coupling to the other parameters."""
    w = 1.3
    c = 0.1 + v[..., 0]
    return 2.0 / c + c / (2 * w * w) + 1e-3 * np.sum(v[..., 1:] ** 2, axis=-1)


@pytest.mark.parametrize("nv,world", [(1, 2), (63, 2), (64, 2), (257, 2), (4096, 3), (5, 4)])
def test_shards_partition_the_grid(nv, world):
    parts = [shard_indices(nv, r, world) for r in range(world)]
    allidx = np.sort(np.concatenate(parts))
    np.testing.assert_array_equal(allidx, np.arange(nv))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 64


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, V, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sw = Sweep(len(V), rank, world, torch.device("cpu"))
        full, am = sw.run(lambda rows: torch.tensor(fake_tau(V[rows]), dtype=torch.float64))
        out_q.put((rank, full.numpy().copy(), int(am)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sweep_matches_serial(world):
    rng = np.random.default_rng(world)
    g = np.geomspace(0.1, 10.0, 23)
    V = np.array([[a, b] for a in g for b in (0.5, 1.0, 2.0)])  # 69 rows: ragged over chunks of 64
    V = np.concatenate([V, V[:5]])  # exact ties: the first occurrence must win
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = fake_tau(V)
    for rank, full, am in res:
        np.testing.assert_array_equal(full, ref)  # bitwise: no arithmetic on the gathered values
        assert am == int(np.argmin(ref))
    _ = rng


def test_single_rank_sweep_no_collective():
    V = np.random.default_rng(0).uniform(0.1, 5.0, (100, 3))
    sw = Sweep(len(V), 0, 1, torch.device("cpu"))
    full, am = sw.run(lambda rows: torch.tensor(fake_tau(V[rows]), dtype=torch.float64))
    np.testing.assert_array_equal(full.numpy(), fake_tau(V))
    assert int(am) == int(np.argmin(fake_tau(V)))


def test_rank_grids_weak_scaling():
    """Weak scaling: world = 1 is the configuration's own grid; for world > 1 every rank gets a grid of
    the same size and the union is the world-fold refined grid (no row shared)."""
    import workloads
    W = workloads.make("c2")
    np.testing.assert_array_equal(workloads.rank_grid(W, 0, 1), W.V)
    for world in (2, 4, 8):
        parts = [workloads.rank_grid(W, r, world) for r in range(world)]
        assert all(p.shape == W.V.shape for p in parts)
        allv = np.concatenate(parts)
        assert len(np.unique(allv, axis=0)) == world * W.nv
        lo, hi = W.V.min(axis=0), W.V.max(axis=0)
        assert np.all(allv >= lo * (1 - 1e-12)) and np.all(allv <= hi * (1 + 1e-12))


def _worker_weak(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nv = 37
        sw = Sweep(nv, rank, world, torch.device("cpu"), scaling="weak")
        V = np.linspace(0.1, 5.0, nv * world).reshape(-1, 1)
        mine = V[rank * nv:(rank + 1) * nv]
        assert np.array_equal(V[sw.mine], mine)  # weak: global rows of this rank
        full, am = sw.run(lambda rows: torch.tensor(fake_tau(V[rows]), dtype=torch.float64))
        out_q.put((rank, full.numpy().copy(), int(am)))
    finally:
        dist.destroy_process_group()


def test_gloo_weak_sweep():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_weak, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    V = np.linspace(0.1, 5.0, 37 * world).reshape(-1, 1)
    ref = fake_tau(V)
    for _, full, am in res:
        np.testing.assert_array_equal(full, ref)
        assert am == int(np.argmin(ref))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_cost_balanced_shards(world):
    """Cost-balanced strong sharding (snake deal of the cost-sorted rows): on c5's 8^4 grid with a
    proxy sum_t |v_t| w_t, every rank's summed cost is within 5 % of the mean (the chunked
    round-robin deal it replaces is far off), and the shards partition the grid with equal sizes."""
    from paper_2312_08201_b200.sweep import shard_balance
    import workloads
    W = workloads.make("c5")
    cost = np.abs(W.V) @ np.array([1.0, 0.7, 1.3, 0.9])
    parts = [shard_indices(W.nv, r, world, cost=cost) for r in range(world)]
    np.testing.assert_array_equal(np.sort(np.concatenate(parts)), np.arange(W.nv))
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    assert shard_balance(W.nv, world, cost) <= 1.05
    assert shard_balance(W.nv, world, cost, balanced=False) > 1.05  # the old chunked deal


def _worker_cost(rank, world, port, V, cost, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sw = Sweep(len(V), rank, world, torch.device("cpu"), cost=cost)
        full, am = sw.run(lambda rows: torch.tensor(fake_tau(V[rows]), dtype=torch.float64))
        out_q.put((rank, full.numpy().copy(), int(am)))
    finally:
        dist.destroy_process_group()


def test_gloo_cost_balanced_sweep_matches_serial():
    world = 3
    V = np.random.default_rng(3).uniform(0.05, 5.0, (301, 2))
    V = np.concatenate([V, V[:4]])  # ties: the first occurrence must win
    cost = V.sum(1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cost, args=(r, world, port, V, cost, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = fake_tau(V)
    for _, full, am in res:
        np.testing.assert_array_equal(full, ref)
        assert am == int(np.argmin(ref))
