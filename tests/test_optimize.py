"""NEXT row f3: batched multi-start Nelder-Mead (host bookkeeping, objective from the engine).

CPU: the Nelder-Mead logic against analytic objectives with known minimisers (the 1-DOF closed form
of tests/golden/one_dof.json's derivation: v* = 2 w (1 - alpha) / phi^2).  GPU: the same on the
real engine, and multi-start on c1 against the oracle-checked grid."""
import numpy as np
import pytest

from paper_2312_08201_b200.optimize import nelder_mead

W_, A_, PHI_ = 1.3, 0.02, 0.7


def one_dof_trace(v):
    c = 2 * A_ * W_ + v * PHI_ ** 2
    return 2.0 / c + c / (2.0 * W_ ** 2)


class Analytic:
    def __init__(self, fn):
        self.fn, self.calls = fn, 0

    def trace_batch(self, V):
        self.calls += 1
        return np.array([self.fn(v) for v in np.atleast_2d(V)])


def test_nm_one_dof_closed_form_argmin():
    prob = Analytic(lambda v: one_dof_trace(v[0]))
    res = nelder_mead(prob, np.log([[0.1], [10.0], [300.0]]), tol_x=1e-8, tol_f=1e-12)
    vstar = 2 * W_ * (1 - A_) / PHI_ ** 2
    assert np.allclose(res.v[:, 0], vstar, rtol=1e-6)
    assert res.f[res.best] == pytest.approx(one_dof_trace(vstar), rel=1e-12)
    assert res.batches == prob.calls and res.evaluations >= 3 * res.iterations.max()


def test_nm_separable_multistart_batches_every_stage():
    """k = 3 separable objective (sum of 1-DOF terms with different optima): every run converges to
    the same minimiser; one engine call per stage carries all runs."""
    ws, phis = np.array([0.7, 1.3, 2.1]), np.array([0.9, 0.5, 1.2])

    def fn(v):
        c = 2 * A_ * ws + v * phis ** 2
        return float(np.sum(2.0 / c + c / (2.0 * ws ** 2)))

    prob = Analytic(fn)
    x0 = np.log(np.array([[0.1, 0.1, 0.1], [50, 50, 50], [0.1, 50, 3], [3, 0.2, 80]], dtype=float))
    res = nelder_mead(prob, x0, tol_x=1e-7, tol_f=1e-12, max_iter=2000)
    vstar = 2 * ws * (1 - A_) / phis ** 2
    np.testing.assert_allclose(res.v, np.broadcast_to(vstar, res.v.shape), rtol=1e-4)
    assert prob.calls < res.evaluations  # batched: fewer calls than evaluations


@pytest.mark.gpu
def test_nm_on_engine_matches_closed_form_and_grid():
    from paper_2312_08201_b200 import Problem

    import oracle
    import workloads
    A0 = np.array([[0.0, W_], [-W_, -2 * A_ * W_]])
    B = np.array([[0.0], [PHI_]])
    P = Problem(A0, B, B, np.eye(2), np.eye(2))
    res = nelder_mead(P, np.log([[0.1], [50.0]]), tol_x=1e-9, tol_f=1e-13)
    vstar = 2 * W_ * (1 - A_) / PHI_ ** 2
    np.testing.assert_allclose(res.v[:, 0], vstar, rtol=1e-5)
    # c1: multi-start from the grid corners; the best run beats (or ties) every grid point
    W = workloads.make("c1")
    P1 = Problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    grid = P1.trace_batch(W.V)
    x0 = np.log(W.V[W.corner_indices()])
    r1 = nelder_mead(P1, x0)
    assert r1.f[r1.best] <= grid.min() * (1 + 1e-4)
    ref = oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, r1.v[r1.best])
    assert r1.f[r1.best] == pytest.approx(ref, rel=1e-9)


def _nm_worker(rank, world, port, out_q):
    import os

    import torch.distributed as dist

    from paper_2312_08201_b200.optimize import nelder_mead_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = Analytic(lambda v: one_dof_trace(v[0]))
        x0 = np.log([[0.1], [10.0], [300.0], [2.0], [0.5]])
        res = nelder_mead_sharded(prob, x0, rank, world, tol_x=1e-8, tol_f=1e-12)
        out_q.put((rank, res.v.copy(), res.f.copy(), res.best))
    finally:
        dist.destroy_process_group()


def test_nm_sharded_multistart_gloo():
    """Multi-start sharded over 2 ranks (gloo): every rank returns the full (f, v) of all starts in
    start order, identical to the serial multi-start run, and the same best start."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x0 = np.log([[0.1], [10.0], [300.0], [2.0], [0.5]])
    ser = nelder_mead(Analytic(lambda v: one_dof_trace(v[0])), x0, tol_x=1e-8, tol_f=1e-12)
    for _, v, f, best in res:
        # each start's run is the same deterministic sequence as in the serial multi-start
        np.testing.assert_allclose(v, ser.v, rtol=1e-12)
        np.testing.assert_allclose(f, ser.f, rtol=1e-12)
        assert best == ser.best


@pytest.mark.gpu
def test_nm_solution_recycling_cuts_applies():
    """Solution recycling between consecutive iterates (lyap_trace_batch_x): each trial point starts
    from its simplex's best vertex; the optimum is unchanged and the T-applications drop."""
    from paper_2312_08201_b200 import Problem

    import workloads
    W = workloads.make("c1")
    P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    x0 = np.log(W.V[W.corner_indices()])
    P.reset_stats()
    plain = nelder_mead(P, x0, tol_x=1e-8, tol_f=1e-12)
    a_plain = P.stats["k1_vectors"]
    P.reset_stats()
    rec = nelder_mead(P, x0, tol_x=1e-8, tol_f=1e-12, recycle=True)
    a_rec = P.stats["k1_vectors"]
    assert rec.f[rec.best] == pytest.approx(plain.f[plain.best], rel=1e-8)
    assert a_rec < 0.9 * a_plain, (a_rec, a_plain, rec.evaluations, plain.evaluations)
    # the engine's graph is updated in place across the many small calls (no re-instantiation)
    assert P.stats["graph_updates"] > 0
