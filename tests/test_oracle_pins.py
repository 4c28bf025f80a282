"""Pins for the CPU oracle (oracle/), independent of the oracle's own formulas.

Each test fixes the oracle against something other than itself: a closed form derived by hand,
the paper's / SPEC's worked values, a brute-force Kronecker solve, a second LAPACK route, or an
invariant the mathematics guarantees.  All CPU (`-m "not gpu"`).
"""
import json
import pathlib

import numpy as np
import pytest
import scipy.linalg

import oracle
import oracle.bartels_stewart as bs
import workloads

GOLDEN = pathlib.Path(__file__).parent / "golden"


# ---------------------------------------------------------------- closed forms (reading R1)
def one_dof_trace(omega, c):
    """1-DOF oscillator A=[[0,w],[-w,-c]], Q=I: X=[[1/c+c/(2w^2), -1/(2w)],[-1/(2w), 1/c]]."""
    return 2.0 / c + c / (2.0 * omega**2)


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())


def test_one_dof_closed_form_golden():
    """tests/golden/one_dof.json: hand-derived values (R1, corrects PAPER.md:853-858)."""
    g = load_golden("one_dof.json")
    for case in g["cases"]:
        w, a, phi, v = case["omega"], case["alpha"], case["phi"], case["v"]
        A0 = np.array([[0.0, w], [-w, -2 * a * w]])
        B = np.array([[0.0], [phi]])
        tau, d = oracle.trace_EX(A0, B, B, np.eye(2), np.eye(2), [v], diagnostics=True)
        assert tau == pytest.approx(case["trace"], rel=1e-13)
        X = d["X"]
        c = 2 * a * w + v * phi**2
        assert X[0, 0] == pytest.approx(1 / c + c / (2 * w * w), rel=1e-13)
        assert X[0, 1] == pytest.approx(-1 / (2 * w), rel=1e-13)
        assert X[1, 1] == pytest.approx(1 / c, rel=1e-13)


def test_uncoupled_modes_block_closed_form():
    """m uncoupled modes in modal phase-space order [q; q'], one damper per mode (P1 blockwise)."""
    rng = np.random.default_rng(7)
    m = 5
    omega = np.sort(rng.uniform(0.5, 4.0, m))
    alpha = 0.03
    phi = rng.uniform(0.3, 1.5, m)
    n = 2 * m
    A0 = np.zeros((n, n))
    A0[:m, m:] = np.diag(omega)
    A0[m:, :m] = -np.diag(omega)
    A0[m:, m:] = -2 * alpha * np.diag(omega)
    B = np.zeros((n, m))
    for t in range(m):
        B[m + t, t] = phi[t]
    sel = np.array([1, 1, 0, 1, 0])  # E = selector of some modes in both blocks
    E = np.diag(np.concatenate([sel, sel]).astype(float))
    for _ in range(5):
        v = rng.uniform(0.01, 20.0, m)
        c = 2 * alpha * omega + v * phi**2
        expect = float(np.sum(sel * one_dof_trace(omega, c)))
        assert oracle.trace_EX(A0, B, B, np.eye(n), E, v) == pytest.approx(expect, rel=1e-12)


def test_one_dof_argmin_is_critical_damping():
    """d tau / dc = 0 at c = 2 w  =>  v* = 2 w (1 - alpha) / phi^2 (argmin pin, P1)."""
    w, a, phi = 1.3, 0.02, 0.7
    A0 = np.array([[0.0, w], [-w, -2 * a * w]])
    B = np.array([[0.0], [phi]])
    vstar = 2 * w * (1 - a) / phi**2
    vs = vstar * np.array([0.9, 0.99, 1.0, 1.01, 1.1])
    taus = oracle.trace_batch(A0, B, B, np.eye(2), np.eye(2), vs[:, None])
    assert int(np.argmin(taus)) == 2
    assert taus[2] == pytest.approx(one_dof_trace(w, 2 * w), rel=1e-13)


def test_scalar_case():
    """n=1: A0=-1, B=1, Q=E=1 -> tau(v) = 1/(2(1+v)) (survey P2)."""
    for v in (0.1, 1.0, 3.0, 250.0, -0.5):
        tau = oracle.trace_EX(np.array([[-1.0]]), np.ones((1, 1)), np.ones((1, 1)),
                              np.eye(1), np.eye(1), [v])
        assert tau == pytest.approx(1.0 / (2.0 * (1.0 + v)), rel=1e-15)


def test_spec_worked_examples():
    """SPEC.md:74-75 and :165/:201/:219 worked values (tests/golden/spec_examples.json)."""
    g = load_golden("spec_examples.json")
    for case in g["lyap"]:
        X = oracle.lyap(np.array(case["A"]), np.array(case["Q"]))
        np.testing.assert_allclose(X, np.array(case["X"]), rtol=1e-14, atol=1e-15)
    for case in g["param"]:
        A0, B = np.array(case["A0"]), np.array(case["B"])
        tau, d = oracle.trace_EX(A0, B, B, np.array(case["Q"]), np.array(case["E"]), case["v"],
                                 diagnostics=True)
        assert tau == pytest.approx(case["trace"], rel=1e-14)
        np.testing.assert_allclose(d["X"], np.array(case["X"]), rtol=1e-14, atol=1e-15)


# ------------------------------------------------------------------ brute force (P3)
def kron_lyap(A, Q):
    """(I (x) A + A (x) I) vec(X) = -vec(Q), dense LU, column-major vec."""
    n = A.shape[0]
    K = np.kron(np.eye(n), A) + np.kron(A, np.eye(n))
    x = np.linalg.solve(K, -Q.reshape(-1, order="F"))
    return x.reshape(n, n, order="F")


@pytest.mark.parametrize("leaf", [1, 2, 3, 5, 64])
def test_kronecker_brute_force(monkeypatch, leaf):
    """50 random stable non-normal instances, n <= 12, k=1..4, Bl != Br; the recursion is
    exercised by shrinking the dtrsyl leaf size so every split branch runs."""
    monkeypatch.setattr(bs, "LEAF", leaf)
    rng = np.random.default_rng(100 + leaf)
    worst = 0.0
    for trial in range(50):
        n = int(rng.integers(1, 13))
        k = int(rng.integers(1, 5))
        A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng, same_b=(trial % 3 == 0))
        v = rng.uniform(0.05, 2.0, k)
        A = oracle.form_A(A0, Bl, Br, v)
        if np.max(np.linalg.eigvals(A).real) >= -1e-3:
            continue
        Xk = kron_lyap(A, Q)
        tau, d = oracle.trace_EX(A0, Bl, Br, Q, E, v, diagnostics=True)
        err = np.linalg.norm(d["X"] - Xk) / np.linalg.norm(Xk)
        worst = max(worst, err)
        assert tau == pytest.approx(np.trace(E @ Xk), rel=1e-11, abs=1e-13)
    assert worst < 1e-12


def test_form_A_against_rank_one_sum():
    """A(v) = A0 + sum_i v_i A_i with A_i = -b_l^i (b_r^i)^T."""
    rng = np.random.default_rng(3)
    A0, Bl, Br, _, _ = workloads.random_stable(9, 3, rng)
    v = rng.standard_normal(3)
    A = A0.copy()
    for i in range(3):
        A -= v[i] * np.outer(Bl[:, i], Br[:, i])
    np.testing.assert_allclose(oracle.form_A(A0, Bl, Br, v), A, rtol=0, atol=1e-15)


# ------------------------------------------------------------ second opinion + invariants
def test_scipy_second_opinion_c1_corners():
    W = workloads.make("c1")
    for i in W.corner_indices():
        A = oracle.form_A(W.A0, W.Bl, W.Br, W.V[i])
        X2 = scipy.linalg.solve_continuous_lyapunov(A, -W.Q)
        tau = oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[i])
        assert tau == pytest.approx(float(np.sum(W.E * X2)), rel=1e-12)


def test_invariants_c1_corners():
    """Symmetry, scale-aware residual (reading R19), backward error, X > 0 for Q = I."""
    W = workloads.make("c1")
    for i in W.corner_indices():
        _, d = oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[i], diagnostics=True)
        assert d["symmetry"] <= 1e-13
        assert d["backward_error"] <= 1e-14
        assert d["residual"] <= max(1e-12, d["floor"])
        assert d["lambda_min_rel"] > 0.0


def test_symmetric_multi_agent_closed_form():
    """Skew part of S set to 0 => A(v) symmetric => X = -A(v)^{-1}/2 for Q = I (survey P5)."""
    rng = np.random.default_rng(11)
    N, d = 25, 3
    S = -0.5 * np.eye(d)
    Adj = np.triu(rng.random((N, N)) < 0.3, 1)
    Adj = (Adj | Adj.T).astype(float)
    LG = np.diag(Adj.sum(1)) - Adj
    A0 = np.kron(np.eye(N), S) - 0.5 * np.kron(LG, np.eye(d))
    e1 = np.eye(d)[0]
    B = np.stack([np.kron(np.eye(N)[0] - np.eye(N)[7], e1), np.kron(np.eye(N)[3] - np.eye(N)[19], e1)], 1)
    E = np.kron(np.eye(N) - np.ones((N, N)) / N, np.outer(e1, e1))
    for v in ([0.3, 2.0], [4.0, 0.05]):
        A = oracle.form_A(A0, B, B, v)
        expect = -0.5 * np.trace(E @ np.linalg.inv(A))
        assert oracle.trace_EX(A0, B, B, np.eye(N * d), E, v) == pytest.approx(expect, rel=1e-12)


def test_small_v_limit_and_sign_flip_invariance():
    """tau(v) -> trace(E X0) as v -> 0+ (SPEC.md:470); flipping a mode-shape sign leaves tau
    unchanged (diag(+-1) similarity, reading R6)."""
    W = workloads.make("c1")
    X0 = scipy.linalg.solve_continuous_lyapunov(W.A0, -W.Q)  # independent LAPACK route
    t0 = float(np.sum(W.E * X0))
    t_small = oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, [1e-9, 1e-9])
    assert t_small == pytest.approx(t0, rel=1e-7)
    m = W.n // 2
    B2 = W.Bl.copy()
    B2[m + 3] *= -1
    v = W.V[77]
    a = oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, v)
    b = oracle.trace_EX(W.A0, B2, B2, W.Q, W.E, v)
    assert a == pytest.approx(b, rel=1e-12)


def test_golden_config_traces_subset():
    """Re-run the oracle on a few stored config samples (tools/make_golden.py output)."""
    for name, count in (("c1", 6), ("c3", 1)):
        g = load_golden(f"oracle_{name}.json")
        W = workloads.make(name)
        for idx, tau in list(zip(g["indices"], g["traces"]))[:count]:
            assert oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[idx]) == pytest.approx(tau, rel=1e-12)


# ----------------------------------------------------------------------------- stability filter (f4)
def test_stability_oracle_one_dof_closed_form():
    """Rightmost eigenvalue of A(v) = [[0, w], [-w, -c]], c = 2 a w + v phi^2 (PAPER.md:1183 filter):
    Re = -c/2 below critical damping, (-c + sqrt(c^2 - 4 w^2))/2 above; stable iff c > 0."""
    w, a, phi = 1.3, 0.02, 0.7
    A0 = np.array([[0.0, w], [-w, -2 * a * w]])
    B = np.array([[0.0], [phi]])
    for v in (-3.0, -0.2, -2 * a * w / phi ** 2 * 1.001, -2 * a * w / phi ** 2 * 0.999, 0.0, 0.5, 7.0, 40.0):
        c = 2 * a * w + v * phi ** 2
        expect = -c / 2 if c * c < 4 * w * w else (-c + np.sqrt(c * c - 4 * w * w)) / 2
        got = oracle.rightmost_real_part(A0, B, B, [v])
        assert got == pytest.approx(expect, abs=1e-12 * max(1.0, abs(c)))
        assert oracle.stable_mask(A0, B, B, [[v]])[0] == (c > 0)
        assert oracle.unstable_count(A0, B, B, [v]) == (2 if c < 0 else 0)  # both roots cross together


def test_stability_oracle_diagonal_rank_one():
    """A0 = diag(d), Bl = Br = e_1: A(v) = diag(d_1 - v, d_2, ...), so the rightmost real part is
    max(d_1 - v, d_2, ...) exactly."""
    d = np.array([-0.5, -2.0, -3.5, -0.75])
    A0 = np.diag(d)
    e1 = np.zeros((4, 1))
    e1[0] = 1.0
    for v in (-1.0, -0.5, -0.25, 0.0, 0.1, 5.0):
        assert oracle.rightmost_real_part(A0, e1, e1, [v]) == pytest.approx(max(d[0] - v, d[1], d[2], d[3]), abs=1e-14)
    np.testing.assert_array_equal(oracle.stable_mask(A0, e1, e1, [[-1.0], [-0.5], [0.2]]), [False, False, True])


def test_stability_oracle_quadratic_formula():
    """Random 2 x 2 A(v): eigenvalues from the characteristic polynomial l^2 - tr l + det."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        A0 = rng.standard_normal((2, 2))
        Bl, Br = rng.standard_normal((2, 2)), rng.standard_normal((2, 2))
        v = rng.uniform(-2, 2, 2)
        A = A0 - Bl @ np.diag(v) @ Br.T
        tr, det = np.trace(A), np.linalg.det(A)
        disc = complex(tr * tr - 4 * det)
        roots = [(tr + np.sqrt(disc)) / 2, (tr - np.sqrt(disc)) / 2]
        assert oracle.rightmost_real_part(A0, Bl, Br, v) == pytest.approx(max(r.real for r in roots), abs=1e-12)
