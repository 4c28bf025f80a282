"""CPU oracle: trace(E X(v)) by a per-v Bartels-Stewart solve of the full Lyapunov equation.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
`cpu_baseline` / `--impl reference` legs may import or call anything under oracle/.  The
product path (paper_2312_08201_b200/) never imports it and shares no code with it.

What it computes (the plain definition, eqs. (Ljap jdba 1) and (eq:formA)):
for each parameter vector v,

    A(v) = A0 - Bl diag(v) Br^T,        A(v) X + X A(v)^T = -Q,        tau(v) = trace(E X).

How (the naive baseline the paper names: "apply the Bartels-Stewart algorithm
to each instance"), step by step, in float64:

  1. form A(v) explicitly;
  2. real Schur form A = U T U^T (LAPACK dgees through scipy.linalg.schur; T quasi upper
     triangular with 1x1 / 2x2 diagonal blocks);
  3. C = -U^T Q U;
  4. solve T Y + Y T^T = C by back substitution over the diagonal blocks, organised as the
     recursive blocked form of the same recurrence (split T without cutting a 2x2 block,
     solve the trailing part, update the leading right-hand side with one GEMM, recurse),
     with LAPACK dtrsyl (the textbook block recurrence) at leaves of order <= LEAF;
     every block of Y is computed -- symmetry is NOT exploited so it stays a check;
  5. X = U Y U^T;
  6. tau = sum_ij E_ij X_ij, plus diagnostics (residual, normwise backward error in the
     normalisation of Prop. 2.1, symmetry, smallest eigenvalue).

The second, independent route used only as a cross-check in tests is
scipy.linalg.solve_continuous_lyapunov (LAPACK trsyl unblocked).

Pins (tests/test_oracle_pins.py, all `-m "not gpu"`): the 1-DOF damped-oscillator closed
form (reading R1, correcting PAPER.md:853-858), the n=1 scalar case, SPEC's n=2
worked example, a brute-force Kronecker solve for n <= 12 on random non-normal A, the
symmetric multi-agent closed form X = -A^{-1}/2, and the invariants (symmetry, residual,
positive definiteness, v -> 0 limit, eigenvector-sign invariance).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
from scipy.linalg.lapack import dtrsyl

__all__ = ["form_A", "sylvester_quasi_triangular", "lyap", "trace_EX", "trace_batch", "LEAF"]

LEAF = 64


def form_A(A0: np.ndarray, Bl: np.ndarray, Br: np.ndarray, v) -> np.ndarray:
    """A(v) = A0 - Bl diag(v) Br^T  (eq:formA)."""
    v = np.asarray(v, dtype=np.float64)
    return A0 - (Bl * v[None, :]) @ Br.T


def _split_point(T: np.ndarray) -> int:
    """Half-way split index that does not cut a 2x2 diagonal block of quasi-triangular T."""
    h = T.shape[0] // 2
    if h > 0 and T[h, h - 1] != 0.0:
        h += 1
    return h


def sylvester_quasi_triangular(A: np.ndarray, B: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Solve A Y + Y B^T = C for quasi upper triangular A (p x p) and B (q x q).

    Block back substitution (Bartels & Stewart) in recursive blocked form:
      split A = [[A11, A12], [0, A22]]:  A22 Y2 + Y2 B^T = C2,  A11 Y1 + Y1 B^T = C1 - A12 Y2;
      split B = [[B11, B12], [0, B22]]:  A Y2 + Y2 B22^T = C2,  A Y1 + Y1 B11^T = C1 - Y2 B12^T.
    Leaves (both orders <= LEAF) call LAPACK dtrsyl with op(B) = B^T.
    """
    p, q = A.shape[0], B.shape[0]
    if p == 0 or q == 0:
        return np.zeros((p, q))
    ha = _split_point(A) if p > LEAF else 0
    hb = _split_point(B) if q > LEAF else 0
    split_a = 0 < ha < p
    split_b = 0 < hb < q
    if not split_a and not split_b:
        Y, scale, info = dtrsyl(A, B, C, trana="N", tranb="T", isgn=1)
        if info < 0:
            raise RuntimeError(f"dtrsyl illegal argument {-info}")
        # info == 1: A and -B have close eigenvalues; result perturbed (reported by residual)
        return Y / scale
    if split_a and (p >= q or not split_b):
        h = ha
        Y2 = sylvester_quasi_triangular(A[h:, h:], B, C[h:, :])
        Y1 = sylvester_quasi_triangular(A[:h, :h], B, C[:h, :] - A[:h, h:] @ Y2)
        return np.vstack([Y1, Y2])
    h = hb
    Y2 = sylvester_quasi_triangular(A, B[h:, h:], C[:, h:])
    Y1 = sylvester_quasi_triangular(A, B[:h, :h], C[:, :h] - Y2 @ B[:h, h:].T)
    return np.hstack([Y1, Y2])


def lyap(A: np.ndarray, Q: np.ndarray) -> np.ndarray:
    """X solving A X + X A^T = -Q (Bartels-Stewart; steps 2-5 of the module docstring)."""
    T, U = scipy.linalg.schur(A, output="real")
    C = -(U.T @ Q @ U)
    Y = sylvester_quasi_triangular(T, T, C)
    return U @ Y @ U.T


def trace_EX(A0, Bl, Br, Q, E, v, diagnostics: bool = False):
    """tau(v) = trace(E X(v)); optionally with the invariant diagnostics."""
    A = form_A(A0, Bl, Br, v)
    X = lyap(A, Q)
    tau = float(np.sum(E * X.T))  # trace(E X) = sum_ij E_ij X_ji
    if not diagnostics:
        return tau
    R = A @ X + X @ A.T + Q
    nR = np.linalg.norm(R)
    nQ = np.linalg.norm(Q)
    nX = np.linalg.norm(X)
    nA = np.linalg.norm(A)
    Xs = 0.5 * (X + X.T)
    lam = np.linalg.eigvalsh(Xs)
    return tau, {
        "residual": nR / nQ,
        "backward_error": nR / (2 * nA * nX + nQ),
        "floor": 100 * np.finfo(float).eps * (2 * nA * nX + nQ) / nQ,
        "symmetry": np.linalg.norm(X - X.T) / nX,
        "lambda_min_rel": lam[0] / max(abs(lam[-1]), 1e-300),
        "X": X,
    }


def trace_batch(A0, Bl, Br, Q, E, V) -> np.ndarray:
    """Oracle traces for every row of V (one Bartels-Stewart solve per row)."""
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    return np.array([trace_EX(A0, Bl, Br, Q, E, v) for v in V])
