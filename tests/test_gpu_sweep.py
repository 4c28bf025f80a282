"""M1 (all-gather + argmin) and the sharded sweep on the real CUDA engine (north star (c), SURVEY §8(e),
§4.2 item 5; VERDICT r1 'Next round' item 1).  The argmin is pinned twice: against the oracle's golden
traces of the whole c1 grid, and against the closed-form critical-damping minimiser of a 1-DOF chain
(from PAPER.md:748-757, 816-834)."""
import json
import pathlib

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu
GOLDEN = pathlib.Path(__file__).parent / "golden"
RTOL = 1e-9


def _problem(*args, **kw):
    from paper_2312_08201_b200 import Problem
    return Problem(*args, **kw)


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


def _golden(name):
    return json.loads((GOLDEN / f"oracle_{name}.json").read_text())


# ----------------------------------------------------------------------------- M1 (argmin) on the engine
def test_sweep_argmin_c1_matches_oracle_golden():
    """M1: the engine's traces of the whole c1 grid through Sweep.run (the bench's step) give the
    oracle's argmin (tests/golden/oracle_c1.json holds all 256 oracle traces; flat index 204)."""
    import torch
    from paper_2312_08201_b200.sweep import Sweep
    g = _golden("c1")
    assert g["indices"] == list(range(256))
    W = workloads.make("c1")
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    Vd = torch.tensor(W.V, device="cuda")
    sw = Sweep(W.nv, 0, 1, torch.device("cuda"))
    full, am = sw.run(lambda rows: P.trace_batch(Vd[torch.as_tensor(rows, device="cuda")]))
    ref = np.array(g["traces"])
    assert int(am) == int(np.argmin(ref)) == 204
    assert rel_err(full.cpu().numpy(), ref).max() <= RTOL
    P.close()


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_sweep_argmin_over_golden_sample(name):
    """M1 on the 256-point golden samples of c2/c3: the engine's argmin over the sampled rows is the
    oracle's (unique minimum: the two smallest oracle traces differ by far more than RTOL)."""
    import torch
    from paper_2312_08201_b200.sweep import Sweep
    g = _golden(name)
    W = workloads.make(name)
    idx = np.array(g["indices"])
    ref = np.array(g["traces"])
    srt = np.sort(ref)
    assert (srt[1] - srt[0]) / abs(srt[0]) > 100 * RTOL  # the minimiser is well separated
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    Vd = torch.tensor(W.V[idx], device="cuda")
    sw = Sweep(len(idx), 0, 1, torch.device("cuda"))
    full, am = sw.run(lambda rows: P.trace_batch(Vd[torch.as_tensor(rows, device="cuda")]))
    assert int(am) == int(np.argmin(ref))
    assert rel_err(full.cpu().numpy(), ref).max() <= RTOL
    P.close()


def test_sweep_argmin_one_dof_critical_damping():
    """M1 pinned by a closed form: one mode A0 = [[0, w], [-w, -2 a w]], damper weight phi:
    tau(v) = 2/c + c/(2 w^2), c = 2 a w + v phi^2, minimised at critical damping c = 2w, i.e.
    v* = 2 w (1 - a) / phi^2.  The engine's argmin over a fine grid is the grid point nearest v*."""
    import torch
    from paper_2312_08201_b200.sweep import Sweep
    w, a, phi = 1.7, 0.02, 0.6
    A0 = np.array([[0.0, w], [-w, -2 * a * w]])
    B = np.array([[0.0], [phi]])
    V = np.geomspace(0.5, 50.0, 2001)[:, None]
    P = _problem(A0, B, B, np.eye(2), np.eye(2))
    sw = Sweep(len(V), 0, 1, torch.device("cuda"))
    Vd = torch.tensor(V, device="cuda")
    full, am = sw.run(lambda rows: P.trace_batch(Vd))
    c = 2 * a * w + V[:, 0] * phi ** 2
    closed = 2.0 / c + c / (2 * w * w)
    assert rel_err(full.cpu().numpy(), closed).max() <= 1e-11
    vstar = 2 * w * (1 - a) / phi ** 2
    assert int(am) == int(np.argmin(np.abs(np.log(V[:, 0] / vstar))))
    P.close()


# ----------------------------------------------------------------------------- boundary / scheduling
def test_device_schedule_matches_unscheduled_and_regq_growth():
    """Device-side scheduling (sched.cuh: cost keys + CUB radix sort + regime map) only permutes the
    work; a recycle-regime map that must grow between calls (small nv, then a larger nv on one ctx)
    keeps parity (regq capacity)."""
    import torch
    W = workloads.make("c1")
    ref = np.array(_golden("c1")["traces"])
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    P.build_recycle(V=W.V, s=16)
    small = P.trace_batch(torch.tensor(W.V[:5], device="cuda")).cpu().numpy()
    assert rel_err(small, ref[:5]).max() <= RTOL
    full = P.trace_batch(torch.tensor(W.V, device="cuda")).cpu().numpy()
    assert rel_err(full, ref).max() <= RTOL
    P.close()
    plain = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, schedule=False)
    assert rel_err(plain.trace_batch(W.V), ref).max() <= RTOL
    plain.close()


def test_trace_batch_rejects_bad_device_shape():
    import torch
    W = workloads.make("c1")
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    with pytest.raises(ValueError):
        P.trace_batch(torch.zeros(4, 3, dtype=torch.float64, device="cuda"))
    P.close()


# ----------------------------------------------------------------------------- sharded sweep, real engine
def _sharded_worker(rank, world, port, name, mixed, out_q):
    import os

    import torch
    import torch.distributed as dist
    from paper_2312_08201_b200 import Problem
    from paper_2312_08201_b200.sweep import Sweep
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = workloads.make(name)
        P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E, device=0, recycle=0, mixed=mixed)
        sw = Sweep(W.nv, rank, world, torch.device("cpu"), scaling="strong", cost=P.cost_proxy(W.V))
        full, am = sw.run(lambda rows: torch.tensor(P.trace_batch(W.V[rows])))
        out_q.put((rank, full.numpy().copy(), int(am)))
        P.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,mixed", [("c1", 0), ("c2", 0), ("c1", 1)])
def test_sharded_sweep_real_engine(name, mixed):
    """two ranks (gloo, both on cuda:0) running the real engine on their cost-balanced
    shards against a single-rank run of the whole grid.  FP64 engine, recycling off: BITWISE (every v
    starts from x = 0 and every reduction has a fixed order, so a trace does not depend on the batch it
    was solved in).  Mixed precision: bitwise equality across batches is not claimed
    (refinement cycles end on thresholds): <= 1e-10 relative, same argmin."""
    import socket

    import torch.multiprocessing as mp
    W = workloads.make(name)
    P1 = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, recycle=0, mixed=mixed)
    single = P1.trace_batch(W.V)
    P1.close()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, name, mixed, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, full, am in res:
        if mixed:
            assert rel_err(full, single).max() <= 1e-10
        else:
            np.testing.assert_array_equal(full, single)
        assert am == int(np.argmin(single))
