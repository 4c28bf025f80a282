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


def nelder_mead(problem, x0_log: np.ndarray, *, step: float = 0.5, tol_x: float = 1e-4, tol_f: float = 1e-4,
                max_iter: int = 400) -> NMResult:
    """Batched Nelder-Mead on f(v) = trace(E X(v)), v = exp(x).  x0_log: (starts, k) initial points."""
    X0 = np.atleast_2d(np.asarray(x0_log, dtype=np.float64))
    S, k = X0.shape
    state = {"evals": 0, "batches": 0}

    def f(xlog: np.ndarray) -> np.ndarray:
        if xlog.size == 0:
            return np.zeros(0)
        state["evals"] += xlog.shape[0]
        state["batches"] += 1
        return np.asarray(problem.trace_batch(np.exp(xlog)), dtype=np.float64)

    # initial simplexes: x0 and x0 + step * e_j
    simp = np.repeat(X0[:, None, :], k + 1, axis=1)
    for j in range(k):
        simp[:, j + 1, j] += step
    fv = f(simp.reshape(-1, k)).reshape(S, k + 1)
    active = np.ones(S, dtype=bool)
    iters = np.zeros(S, dtype=np.int64)
    for _ in range(max_iter):
        order = np.argsort(fv, axis=1, kind="stable")
        simp = np.take_along_axis(simp, order[:, :, None], axis=1)
        fv = np.take_along_axis(fv, order, axis=1)
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
        if need2.any():
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
        if shrink.any():
            B = A[shrink]
            simp[B, 1:] = simp[B, :1] + 0.5 * (simp[B, 1:] - simp[B, :1])
            fv[B, 1:] = f(simp[B, 1:].reshape(-1, k)).reshape(len(B), k)
    order = np.argsort(fv, axis=1, kind="stable")
    simp = np.take_along_axis(simp, order[:, :, None], axis=1)
    fv = np.take_along_axis(fv, order, axis=1)
    best = int(np.argmin(fv[:, 0]))
    return NMResult(v=np.exp(simp[:, 0]), f=fv[:, 0].copy(), iterations=iters, evaluations=state["evals"],
                    batches=state["batches"], best=best)
