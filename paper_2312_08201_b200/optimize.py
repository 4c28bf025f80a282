"""NEXT row f3: optimizer-driven sequences of parameter vectors.

The paper's Example 1 minimises the total average energy trace(X(v)) over damper viscosities with
MATLAB `fminsearch` (Nelder-Mead, tolerance 1e-4).  A single Nelder-Mead
run evaluates one or two v at a time -- latency-bound on a GPU.  Here many simplexes run at once
(multi-start; `starts` rows) and every stage of a step (reflection, then expansion or contraction,
then shrink) evaluates the trial points of ALL simplexes with ONE lyap_trace_batch call, so each GPU
call carries a batch.  Search in log(v) (viscosities are positive; the paper's grids are
log-spaced).  The Nelder-Mead decisions are host bookkeeping on (starts x k) numbers; every
objective value comes from the CUDA engine.

Coefficients: reflection 1, expansion 2, contraction 1/2, shrink 1/2 (Lagarias et al. 1998, the
fminsearch choice); stopping: max |f_i - f_0| <= tol_f and max ||x_i - x_0||_inf <= tol_x per
simplex, as fminsearch's TolFun / TolX (applied in log v).

Recycling between consecutive iterates ("slowly varying" sequences; Alg. 1 remark
PAPER.md:670-671): with `recycle=True` (engine problems) every trial point starts its Krylov solve
from the solution g of its simplex's current best vertex (lyap_trace_batch_x), and every evaluated
vertex keeps its solution on the device.  Near convergence the simplex shrinks, the guesses become
accurate and the solves cheap; the certified result does not depend on the guess.

Multi-GPU (`nelder_mead_sharded`): the starts are dealt round-robin to the ranks, each rank runs its
simplexes on its own GPU, and the (f, v) of every start are all-gathered; the best run is the
smallest f, first start on ties.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class NMResult:
    v: np.ndarray          # (starts, k) best parameter vector of every run
    f: np.ndarray          # (starts,) objective at v
    iterations: np.ndarray  # (starts,)
    evaluations: int       # objective evaluations (all runs)
    batches: int           # lyap_trace_batch calls
    best: int              # index of the best run (smallest f, first on ties)
    applies: int = 0       # T-applications spent by the engine (recycle=True runs; 0 otherwise)


def nelder_mead(problem, x0_log: np.ndarray, *, step: float = 0.5, tol_x: float = 1e-4, tol_f: float = 1e-4,
                max_iter: int = 400, recycle: bool = False) -> NMResult:
    """Batched Nelder-Mead on f(v) = trace(E X(v)), v = exp(x).  x0_log: (starts, k) initial points.
    recycle: warm-start every trial point from its simplex's best vertex (needs Problem.trace_batch_x)."""
    X0 = np.atleast_2d(np.asarray(x0_log, dtype=np.float64))
    S, k = X0.shape
    state = {"evals": 0, "batches": 0, "applies": 0}
    store = {}  # recycle: per simplex, per vertex, the device solution of the vertex

    def f(xlog: np.ndarray, owner=None, guess=None) -> np.ndarray:
        """Objective of the rows of xlog; with recycle, owner[i] = simplex of row i and guess = the
        solutions to start from (or None).  Returns values (and the solutions when recycling)."""
        if xlog.size == 0:
            return (np.zeros(0), None) if recycle else np.zeros(0)
        state["evals"] += xlog.shape[0]
        state["batches"] += 1
        if not recycle:
            return np.asarray(problem.trace_batch(np.exp(xlog)), dtype=np.float64)
        import torch
        V = torch.tensor(np.exp(xlog), device="cuda")
        tau, G, _st, ap, _rs = problem.trace_batch_x(V, guess, return_diagnostics=True)
        state["applies"] += int(ap.sum().item())
        return tau.cpu().numpy().astype(np.float64), G

    def guesses(owners):
        if not recycle or "G" not in store:
            return None
        import torch
        return store["G"][torch.as_tensor(owners, device=store["G"].device), 0].contiguous()

    # initial simplexes: x0 and x0 + step * e_j
    simp = np.repeat(X0[:, None, :], k + 1, axis=1)
    for j in range(k):
        simp[:, j + 1, j] += step
    if recycle:
        fv, G0 = f(simp.reshape(-1, k))
        fv = fv.reshape(S, k + 1)
        store["G"] = G0.reshape(S, k + 1, *G0.shape[1:]).clone()
    else:
        fv = f(simp.reshape(-1, k)).reshape(S, k + 1)
    active = np.ones(S, dtype=bool)
    iters = np.zeros(S, dtype=np.int64)
    for _ in range(max_iter):
        order = np.argsort(fv, axis=1, kind="stable")
        simp = np.take_along_axis(simp, order[:, :, None], axis=1)
        fv = np.take_along_axis(fv, order, axis=1)
        if recycle:
            import torch
            oi = torch.as_tensor(order, device=store["G"].device)
            store["G"] = store["G"][torch.arange(S, device=oi.device)[:, None], oi]
        conv = (np.max(np.abs(fv[:, 1:] - fv[:, :1]), axis=1) <= tol_f) & \
               (np.max(np.abs(simp[:, 1:] - simp[:, :1]), axis=(1, 2)) <= tol_x)
        active &= ~conv
        if not active.any():
            break
        A = np.nonzero(active)[0]
        iters[A] += 1
        cen = simp[A, :-1].mean(axis=1)
        worst = simp[A, -1]
        xr = cen + (cen - worst)
        if recycle:
            fr, Gr = f(xr, A, guesses(A))
        else:
            fr = f(xr)
        f0, fs, fw = fv[A, 0], fv[A, -2], fv[A, -1]
        accept_r = (fr >= f0) & (fr < fs)
        do_exp = fr < f0
        do_out = (fr >= fs) & (fr < fw)
        do_in = fr >= fw
        xe = cen + 2.0 * (cen - worst)
        xc_out = cen + 0.5 * (xr - cen)
        xc_in = cen + 0.5 * (worst - cen)
        second = np.where(do_exp[:, None], xe, np.where(do_out[:, None], xc_out, xc_in))
        need2 = ~accept_r
        f2 = np.full(len(A), np.inf)
        G2 = None
        if need2.any():
            if recycle:
                f2[need2], G2 = f(second[need2], A[need2], guesses(A[need2]))
            else:
                f2[need2] = f(second[need2])
        new_x, new_f = worst.copy(), fw.copy()
        # reflection accepted
        new_x[accept_r], new_f[accept_r] = xr[accept_r], fr[accept_r]
        # expansion: keep the better of expansion and reflection
        e_better = do_exp & (f2 < fr)
        e_worse = do_exp & ~(f2 < fr)
        new_x[e_better], new_f[e_better] = second[e_better], f2[e_better]
        new_x[e_worse], new_f[e_worse] = xr[e_worse], fr[e_worse]
        # contractions
        c_out_ok = do_out & (f2 <= fr)
        c_in_ok = do_in & (f2 < fw)
        c_ok = c_out_ok | c_in_ok
        new_x[c_ok], new_f[c_ok] = second[c_ok], f2[c_ok]
        shrink = (do_out & ~c_out_ok) | (do_in & ~c_in_ok)
        simp[A[~shrink], -1] = new_x[~shrink]
        fv[A[~shrink], -1] = new_f[~shrink]
        if recycle:  # keep the solution of the vertex that replaced the worst one
            import torch
            dev = store["G"].device
            src_r = accept_r | e_worse
            for mask, Gsrc, pos in ((src_r, Gr, np.nonzero(src_r)[0]), (e_better | c_ok, G2, None)):
                if Gsrc is None or not mask.any():
                    continue
                if pos is None:  # G2 rows are the need2 rows, in order
                    rows = np.cumsum(need2) - 1
                    pos = rows[mask]
                store["G"][torch.as_tensor(A[mask], device=dev), -1] = Gsrc[torch.as_tensor(pos, device=dev)]
        if shrink.any():
            B = A[shrink]
            simp[B, 1:] = simp[B, :1] + 0.5 * (simp[B, 1:] - simp[B, :1])
            if recycle:
                import torch
                own = np.repeat(B, k)
                fs_, Gs_ = f(simp[B, 1:].reshape(-1, k), own, guesses(own))
                fv[B, 1:] = fs_.reshape(len(B), k)
                store["G"][torch.as_tensor(B, device=store["G"].device), 1:] = Gs_.reshape(len(B), k, *Gs_.shape[1:])
            else:
                fv[B, 1:] = f(simp[B, 1:].reshape(-1, k)).reshape(len(B), k)
    order = np.argsort(fv, axis=1, kind="stable")
    simp = np.take_along_axis(simp, order[:, :, None], axis=1)
    fv = np.take_along_axis(fv, order, axis=1)
    best = int(np.argmin(fv[:, 0]))
    return NMResult(v=np.exp(simp[:, 0]), f=fv[:, 0].copy(), iterations=iters, evaluations=state["evals"],
                    batches=state["batches"], best=best, applies=state["applies"])


def nelder_mead_sharded(problem, x0_log: np.ndarray, rank: int, world: int, group=None, **kw) -> NMResult:
    """Multi-start Nelder-Mead with the starts dealt round-robin to `world` ranks (one GPU each); the
    (f, v) of every start are all-gathered (torch.distributed), so every rank returns the full result
    in start order.  Counters (iterations, evaluations, batches, applies) are this rank's."""
    import torch
    import torch.distributed as dist
    X0 = np.atleast_2d(np.asarray(x0_log, dtype=np.float64))
    S, k = X0.shape
    mine = np.arange(rank, S, world)
    res = nelder_mead(problem, X0[mine], **kw) if len(mine) else None
    per = (S + world - 1) // world
    buf = torch.full((per, k + 2), float("nan"), dtype=torch.float64)
    if res is not None:
        buf[: len(mine), 0] = torch.tensor(mine, dtype=torch.float64)
        buf[: len(mine), 1] = torch.tensor(res.f)
        buf[: len(mine), 2:] = torch.tensor(res.v)
    if world > 1:
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf, group=group)
        allb = torch.cat(out)
    else:
        allb = buf
    allb = allb[~torch.isnan(allb[:, 0])]
    idx = allb[:, 0].long().numpy()
    f = np.empty(S)
    v = np.empty((S, k))
    f[idx] = allb[:, 1].numpy()
    v[idx] = allb[:, 2:].numpy()
    best = int(np.argmin(f))  # first start on ties
    it = res.iterations if res is not None else np.zeros(0, np.int64)
    return NMResult(v=v, f=f, iterations=it, evaluations=res.evaluations if res else 0,
                    batches=res.batches if res else 0, best=best, applies=res.applies if res else 0)
