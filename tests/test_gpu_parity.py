"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle and independent references.

Tolerance (north star, BASELINE.json): relative error <= 1e-9 in FP64 on every trace.
"""
import json
import pathlib

import numpy as np
import pytest
import scipy.linalg

import oracle
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


# ----------------------------------------------------------------------------- K1 unit test
def _complex_factors(st, n):
    """Full eigen-index complex lambda, B^r, B~l from the exported folded state."""
    npairs = st["n_pairs"]
    lam = st["lam"][:, 0] + 1j * st["lam"][:, 1]
    br = st["bhr"].astype(complex)
    bl = st["btl"].astype(complex)
    for r in range(npairs):
        c = 2 * r
        lam[c + 1] = np.conj(lam[c])
        zr = st["bhr"][c] + 1j * st["bhr"][c + 1]
        zl = st["btl"][c] + 1j * st["btl"][c + 1]
        br[c], br[c + 1] = zr, np.conj(zr)
        bl[c], bl[c + 1] = zl, np.conj(zl)
    return lam, br, bl


def _fold(Gc, npairs, npad):
    k, n = Gc.shape
    X = np.zeros((k, npad))
    for r in range(npairs):
        X[:, 2 * r], X[:, 2 * r + 1] = Gc[:, 2 * r].real, Gc[:, 2 * r].imag
    X[:, 2 * npairs:n] = Gc[:, 2 * npairs:n].real
    return X


def _unfold(X, npairs, n):
    k = X.shape[0]
    G = np.zeros((k, n), complex)
    for r in range(npairs):
        z = X[:, 2 * r] + 1j * X[:, 2 * r + 1]
        G[:, 2 * r], G[:, 2 * r + 1] = z, np.conj(z)
    G[:, 2 * npairs:n] = X[:, 2 * npairs:n]
    return G


@pytest.mark.parametrize("n,k,seed", [(7, 1, 0), (16, 2, 1), (33, 3, 2), (40, 4, 3), (130, 2, 4),
                                      (1600, 2, 5)])  # n > 1536: the 128x128x32 large-tile DMMA configuration
def test_k1_apply_against_paper_blocks(n, k, seed):
    """K1 (folded DMMA GEMM + prologue + epilogue) against the complex operator built entrywise from
    eqs. (N1M1), (N2M1), (N1M2) with the same seed factors."""
    import torch
    rng = np.random.default_rng(seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng)
    P = _problem(A0, Bl, Br, Q, E)
    st = P.export_state()
    npairs, npad = st["n_pairs"], st["npad"]
    lam, br, bl = _complex_factors(st, n)
    L = 1.0 / (lam[:, None] + lam[None, :])
    F = np.einsum("ij,is,it->jst", L, br, bl)  # T_d blocks, eq. (N1M1) / (2,2) block
    # exported F (reps only) agrees with the paper formula
    reps = list(range(0, 2 * npairs, 2)) + list(range(2 * npairs, n))
    Fx = st["F"][..., 0] + 1j * st["F"][..., 1]
    np.testing.assert_allclose(Fx, F[reps], rtol=1e-11, atol=1e-11 * np.abs(F).max())
    nvec = 5
    Xs, sig = [], rng.uniform(-2, 3, (nvec, k))
    Gs = []
    for _ in range(nvec):
        G = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
        G = _unfold(_fold(G, npairs, npad), npairs, n)  # conjugate-symmetric
        Gs.append(G)
        Xs.append(_fold(G, npairs, npad))
    Y = P.apply_C(torch.tensor(np.stack(Xs), device="cuda"), torch.tensor(sig, device="cuda")).cpu().numpy()
    for v in range(nvec):
        G = Gs[v]
        TG = np.einsum("jst,tj->sj", F, G) + np.einsum("jt,ij,is,ti->sj", bl, L, br, G)
        expect = _fold(sig[v][:, None] * G - TG, npairs, npad)
        scale = np.abs(expect).max()
        np.testing.assert_allclose(Y[v], expect, rtol=0, atol=1e-12 * scale)
        assert np.all(Y[v][:, n:] == 0.0)
    P.close()


def test_setup_spectrum_and_t0():
    """Exported eigenvalues = eig(A0); t0 = trace(E X0) with X0 from an independent LAPACK solve."""
    rng = np.random.default_rng(5)
    n, k = 24, 3
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng)
    P = _problem(A0, Bl, Br, Q, E)
    st = P.export_state()
    lam, _, _ = _complex_factors(st, n)
    ref = np.linalg.eigvals(A0)
    key = lambda z: (np.round(z.real, 9), np.round(z.imag, 9))
    np.testing.assert_allclose(np.array(sorted(lam, key=key)), np.array(sorted(ref, key=key)), atol=1e-10)
    X0 = scipy.linalg.solve_continuous_lyapunov(A0, -Q)
    assert P.info["t0"] == pytest.approx(float(np.sum(0.5 * (E + E.T) * X0)), rel=1e-11)
    P.close()


# ----------------------------------------------------------------------------- parity vs oracle
@pytest.mark.parametrize("n,k,seed,same_b", [(1, 1, 0, True), (6, 2, 1, False), (13, 3, 2, False),
                                             (29, 4, 3, True), (40, 1, 4, False), (64, 2, 5, False)])
def test_random_instances_all_v(n, k, seed, same_b):
    rng = np.random.default_rng(50 + seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng, same_b=same_b)
    V = rng.uniform(0.05, 2.0, (37, k))  # ragged batch
    P = _problem(A0, Bl, Br, Q, E, batch=8)
    tau, st, ap, rs = P.trace_batch(V, return_diagnostics=True)
    ref = oracle.trace_batch(A0, Bl, Br, Q, E, V)
    assert np.all(st == 0), (st, rs)
    assert rel_err(tau, ref).max() <= RTOL, rel_err(tau, ref).max()
    assert np.all(rs <= 1e-12)
    P.close()


def test_scalar_closed_form():
    """n = 1: A0 = -1, B = 1, Q = E = 1 -> tau(v) = 1/(2(1+v))."""
    P = _problem(-np.eye(1), np.ones((1, 1)), np.ones((1, 1)), np.eye(1), np.eye(1))
    v = np.array([[0.1], [1.0], [3.0], [250.0], [-0.5]])
    np.testing.assert_allclose(P.trace_batch(v), 1.0 / (2.0 * (1.0 + v[:, 0])), rtol=1e-13)
    P.close()


def test_zero_and_negative_parameters():
    """v_t = 0 means column t absent; negative v allowed."""
    rng = np.random.default_rng(9)
    A0, Bl, Br, Q, E = workloads.random_stable(20, 3, rng, shift=2.0)
    V = np.array([[0.0, 0.5, 1.0], [0.3, 0.0, 0.0], [0.0, 0.0, 0.0], [-0.2, 0.4, -0.1], [1.0, 1.0, 1.0]])
    P = _problem(A0, Bl, Br, Q, E)
    tau = P.trace_batch(V)
    ref = oracle.trace_batch(A0, Bl, Br, Q, E, V)
    assert rel_err(tau, ref).max() <= RTOL
    assert tau[2] == pytest.approx(P.info["t0"], rel=1e-13)
    P.close()


def test_device_path_equals_host_path_and_edge_batches():
    import torch
    W = workloads.make("c1")
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    h = P.trace_batch(W.V[:50])
    d = P.trace_batch(torch.tensor(W.V[:50], device="cuda")).cpu().numpy()
    assert rel_err(d, h).max() <= 1e-12
    assert P.trace_batch(np.zeros((0, 2))).shape == (0,)
    one = P.trace_batch(W.V[7:8])
    assert one[0] == pytest.approx(h[7], rel=1e-11)
    P.close()


def test_warm_start_and_tiny_batch_agree():
    W = workloads.make("c1")
    idx = W.corner_indices()
    a = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, batch=3, warm_start=True).trace_batch(W.V[idx])
    b = _problem(W.A0, W.Bl, W.Br, W.Q, W.E).trace_batch(W.V[idx])
    assert rel_err(a, b).max() <= 1e-10


def _golden(name):
    return json.loads((GOLDEN / f"oracle_{name}.json").read_text())


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_full_batch_vs_oracle_samples(name):
    """Full BASELINE config, whole grid in one trace_batch (the bench launch configuration); the
    oracle traces of tests/golden (tools/make_golden.py: corners + centre + seeded sample)."""
    g = _golden(name)
    W = workloads.make(name)
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    tau, st, ap, rs = P.trace_batch(W.V, return_diagnostics=True)
    idx = np.array(g["indices"])
    err = rel_err(tau[idx], np.array(g["traces"]))
    assert np.all(st == 0), np.nonzero(st)
    assert err.max() <= RTOL, (err.max(), idx[np.argmax(err)])
    assert np.all(np.isfinite(tau))
    P.close()


def test_schedule_does_not_change_results():
    """Cost-ordered scheduling only permutes the work: traces come back in row order of V."""
    W = workloads.make("c1")
    a = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, schedule=True, batch=16).trace_batch(W.V)
    b = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, schedule=False, batch=16).trace_batch(W.V)
    assert rel_err(a, b).max() <= 1e-10
    g = _golden("c1")
    assert rel_err(a[np.array(g["indices"])], np.array(g["traces"])).max() <= RTOL


def test_slot_groups_deterministic():
    """Two slot groups on two streams (b >= 64): results independent of group/slot assignment, so
    repeated runs are bitwise identical and equal to a single-group run to rounding."""
    W = workloads.make("c1")
    P2 = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, batch=128)
    a = P2.trace_batch(W.V)
    b = P2.trace_batch(W.V)
    np.testing.assert_array_equal(a, b)
    c = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, batch=32).trace_batch(W.V)  # one group
    assert rel_err(a, c).max() <= 1e-11


# ----------------------------------------------------------------------------- edge cases
def test_all_real_spectrum():
    """Symmetric A0: every eigenvalue real, no conjugate pairs (n_pairs = 0 folding path)."""
    rng = np.random.default_rng(21)
    n, k = 30, 2
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    A0 = -(G @ G.T) - 0.5 * np.eye(n)
    B = rng.standard_normal((n, k)) / np.sqrt(n)
    Q, E = np.eye(n), np.diag(rng.uniform(0, 1, n))
    P = _problem(A0, B, B, Q, E)
    assert P.info["n_pairs"] == 0
    V = rng.uniform(0.1, 3.0, (19, k))
    assert rel_err(P.trace_batch(V), oracle.trace_batch(A0, B, B, Q, E, V)).max() <= RTOL


def test_kmax_and_asymmetric_E():
    """k = LYAP_KMAX = 8 and a non-symmetric E (only its symmetric part matters, X = X^T)."""
    rng = np.random.default_rng(22)
    n, k = 24, 8
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng, shift=1.5)
    E = E + 0.3 * np.triu(rng.standard_normal((n, n)), 1)
    V = rng.uniform(0.05, 1.0, (11, k))
    P = _problem(A0, Bl, Br, Q, E)
    assert rel_err(P.trace_batch(V), oracle.trace_batch(A0, Bl, Br, Q, E, V)).max() <= RTOL


def test_forced_restarts_still_converge():
    """A short restart length (m_max = 40, below the ~80 iterations c1's hardest corner needs)
    forces several GMRES cycles; restarts re-verify the true residual."""
    W = workloads.make("c1")
    idx = W.corner_indices()
    tau, st, ap, rs = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, max_dim=40, max_restarts=100).trace_batch(
        W.V[idx], return_diagnostics=True)
    g = _golden("c1")
    ref = dict(zip(g["indices"], g["traces"]))
    assert np.all(st == 0) and ap.max() > 42
    assert rel_err(tau, np.array([ref[i] for i in idx])).max() <= RTOL


def test_error_paths():
    from paper_2312_08201_b200 import LyapError
    # purely imaginary pair: lambda + conj(lambda) = 0 -> seed Lyapunov operator singular
    A0 = np.array([[0.0, 1.0], [-1.0, 0.0]])
    B = np.array([[0.0], [1.0]])
    with pytest.raises(LyapError) as ei:
        _problem(A0, B, B, np.eye(2), np.eye(2))
    assert ei.value.code == 5  # LYAP_ESINGULAR
    # nearly defective A0 (eigenvector matrix ill-conditioned) with a strict cond(S) limit
    A1 = np.array([[-1.0, 1e6], [0.0, -1.0 - 1e-9]])
    with pytest.raises(LyapError) as ei:
        _problem(A1, B, B, np.eye(2), np.eye(2), max_cond_S=1e4)
    assert ei.value.code == 4  # LYAP_EEIG
    # a loose tolerance is honoured (fewer applies, still close)
    W = workloads.make("c1")
    tight = _problem(W.A0, W.Bl, W.Br, W.Q, W.E).trace_batch(W.V[:20], return_diagnostics=True)
    loose = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, tol=1e-6).trace_batch(W.V[:20], return_diagnostics=True)
    assert loose[2].sum() < tight[2].sum()
    assert rel_err(loose[0], tight[0]).max() <= 1e-4


# ----------------------------------------------------------------------------- NEXT row f2
@pytest.mark.parametrize("case", ["c1", "c2", "random_mixed", "random_real"])
def test_full_solution_matches_oracle(case):
    """lyap_solution: X(v) elementwise against the oracle's Bartels-Stewart X.
    c2 (n = 800) runs the batched DMMA GEMMs over several 128 x 128 tiles with a ragged padding."""
    rng = np.random.default_rng(31)
    if case in ("c1", "c2"):
        W = workloads.make(case)
        A0, Bl, Br, Q, E = W.A0, W.Bl, W.Br, W.Q, W.E
        V = W.V[W.corner_indices()]
    elif case == "random_mixed":
        A0, Bl, Br, Q, E = workloads.random_stable(23, 3, rng)
        V = rng.uniform(0.1, 2.0, (4, 3))
    else:
        n = 17
        G = rng.standard_normal((n, n)) / np.sqrt(n)
        A0 = -(G @ G.T) - 0.5 * np.eye(n)
        Bl = rng.standard_normal((n, 2)) / np.sqrt(n)
        Br = rng.standard_normal((n, 2)) / np.sqrt(n)
        Q, E = np.eye(n), np.eye(n)
        V = rng.uniform(0.1, 1.0, (3, 2))
    P = _problem(A0, Bl, Br, Q, E)
    X, tau = P.solution(V, return_traces=True)
    for i, v in enumerate(V):
        _, d = oracle.trace_EX(A0, Bl, Br, Q, E, v, diagnostics=True)
        Xo = d["X"]
        assert np.abs(X[i] - Xo).max() <= 1e-9 * np.abs(Xo).max()
        A = oracle.form_A(A0, Bl, Br, v)
        R = A @ X[i] + X[i] @ A.T + Q
        assert np.linalg.norm(R) <= 1e-9 * np.linalg.norm(Q) * max(1.0, np.linalg.norm(X[i]))
        assert tau[i] == pytest.approx(float(np.sum(0.5 * (E + E.T) * X[i])), rel=1e-9)
    P.close()


# ----------------------------------------------------------------------------- NEXT row f4
def test_setup_like_other_configuration():
    """lyap_setup_like: same A0/Q/E, other dampers (different positions and k); equals a fresh setup,
    matches the oracle, survives destruction of the base (shared, reference-counted basis)."""
    import gc
    W = workloads.make("c1")
    m = W.n // 2
    base = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    A0c, B3, _, _, _, _ = workloads.chain(50, 100.0, 0.02, [5, 20, 44], modes_in_E=10)
    np.testing.assert_allclose(A0c, W.A0)
    other = base.like(B3)
    assert other.info["setup_ms"] < base.info["setup_ms"]
    del base
    gc.collect()
    rng = np.random.default_rng(41)
    V = rng.uniform(0.1, 30.0, (12, 3))
    tau = other.trace_batch(V)
    fresh = _problem(W.A0, B3, B3, W.Q, W.E).trace_batch(V)
    assert rel_err(tau, fresh).max() <= 1e-11
    ref = oracle.trace_batch(W.A0, B3, B3, W.Q, W.E, V[:4])
    assert rel_err(tau[:4], ref).max() <= RTOL
    assert m == 50


# ----------------------------------------------------------------------------- recycling
def test_recycle_any_space_keeps_parity():
    """Flexible GMRES with recycled first directions is exact for ANY space: random U (two regimes)
    must give the oracle's traces; the recycled steps spend no T-apply."""
    W = workloads.make("c1")
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    npad, n = P.info["npad"], W.n
    rng = np.random.default_rng(51)
    U = rng.standard_normal((2, 12, W.k, npad))
    U[..., n:] = 0.0
    seeds = np.array([[0.1, 0.1], [100.0, 100.0]])
    P.set_recycle(U, seeds)
    tau, st, ap, rs = P.trace_batch(W.V, return_diagnostics=True)
    g = _golden("c1")
    idx = np.array(g["indices"])
    assert np.all(st == 0)
    assert rel_err(tau[idx], np.array(g["traces"])).max() <= RTOL
    P.set_recycle(np.zeros((0, 1, W.k, npad)), np.zeros((0, W.k)))  # off again
    tau2 = P.trace_batch(W.V)
    assert rel_err(tau2, tau).max() <= 1e-10


def test_recycle_dependent_directions():
    """A space with a repeated and a zero column: the recycled candidate C(v)u is dependent on the
    current basis inside the first s steps (Arnoldi breakdown).  The cycle must still update x with
    the u_i it used, the space is dropped at the next restart, and every trace matches the oracle."""
    W = workloads.make("c1")
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    npad, n = P.info["npad"], W.n
    rng = np.random.default_rng(52)
    U = rng.standard_normal((1, 10, W.k, npad))
    U[..., n:] = 0.0
    U[0, 3] = U[0, 2]  # dependent: breakdown at step 3
    U[0, 6] = 0.0      # (never reached in a cycle that broke down at 3)
    P.set_recycle(U, np.array([[1.0, 1.0]]))
    tau, st, ap, rs = P.trace_batch(W.V, return_diagnostics=True)
    g = _golden("c1")
    idx = np.array(g["indices"])
    assert np.all(st == 0)
    assert rel_err(tau[idx], np.array(g["traces"])).max() <= RTOL
    U2 = U.copy()
    U2[0, 0] = 0.0  # zero first direction: breakdown at step 0
    P.set_recycle(U2, np.array([[1.0, 1.0]]))
    tau2, st2, _, _ = P.trace_batch(W.V, return_diagnostics=True)
    assert np.all(st2 == 0)
    assert rel_err(tau2[idx], np.array(g["traces"])).max() <= RTOL


@pytest.mark.parametrize("name,s,rounds", [("c1", 24, "1"), ("c1", 24, "2"), ("c2", 48, "2")])
def test_recycle_built_spaces_parity_and_savings(name, s, rounds, monkeypatch):
    """lyap_build_recycle from the 2^k grid corners, with (rounds = 2) and without the refinement
    pass: traces still match the oracle samples and the T-applies per v drop."""
    monkeypatch.setenv("LYAP_RECYCLE_ROUNDS", rounds)
    W = workloads.make(name)
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    P.reset_stats()
    P.trace_batch(W.V)
    t0 = P.stats["k1_vectors"]  # T-applications (recycled steps need none)
    P.build_recycle(V=W.V, s=s)
    P.reset_stats()
    tau, st, ap1, rs = P.trace_batch(W.V, return_diagnostics=True)
    t1 = P.stats["k1_vectors"]
    g = _golden(name)
    idx = np.array(g["indices"])
    assert np.all(st == 0)
    assert rel_err(tau[idx], np.array(g["traces"])).max() <= RTOL
    assert t1 < t0, (t0, t1)


# ----------------------------------------------------------------------------- NEXT row f1
@pytest.mark.parametrize("name,nsub", [("c1", 256), ("c2", 40)])
def test_extended_krylov_projection(name, nsub):
    """EKProblem (§2.2, Alg. 1): an approximation controlled by the backward-error target of
    Prop. 2.1.  A returned LYAP_OK certifies bwd <= eps; the trace error against the oracle must then
    scale with eps (forward error <= condition x backward error: <= 1e3 eps here), and shrink as eps
    does."""
    from paper_2312_08201_b200 import EKProblem
    W = workloads.make(name)
    X0 = scipy.linalg.solve_continuous_lyapunov(W.A0, -W.Q)  # seed solution (independent LAPACK)
    t0 = float(np.sum(W.E * X0))
    g = _golden(name)
    idx = np.array(g["indices"])[:nsub]
    ref = np.array(g["traces"])[:nsub]
    errs, info = [], []
    for eps in (1e-6, 1e-10):
        ek = EKProblem(W.A0, W.Bl, W.Br, X0 @ W.Br, W.E, t0, max_dim=W.n)
        tau, dim, bwd = ek.trace_batch(W.V[idx], eps=eps)
        errs.append(rel_err(tau, ref).max())
        info.append((eps, dim, bwd, errs[-1]))
        assert bwd <= eps, info
        assert errs[-1] <= 1e3 * eps, info
        assert (dim % (4 * W.k) == 0 or dim == W.n) and dim <= W.n  # EK blocks, or completed to R^n
        ek.close()
    assert errs[1] <= errs[0], info


@pytest.mark.parametrize("name,nsub,eps", [("c1", 64, 1e-10), ("c3", 48, 1e-10)])
def test_extended_krylov_per_v_certification(name, nsub, eps):
    """Alg. 1 per-v certification: every v's trace comes with its own Prop. 2.1
    backward error <= eps; the traces match the oracle to <= 1e3 eps.  c3 (the multi-agent network,
    the paper's Ex. 2/3 setting: spaces of 8-56 columns) compresses: every v is
    certified with a basis far below n."""
    from paper_2312_08201_b200 import EKProblem
    W = workloads.make(name)
    X0 = scipy.linalg.solve_continuous_lyapunov(W.A0, -W.Q)
    t0 = float(np.sum(0.5 * (W.E + W.E.T) * X0))
    g = _golden(name)
    idx = np.array(g["indices"])[:nsub]
    ref = np.array(g["traces"])[:nsub]
    ek = EKProblem(W.A0, W.Bl, W.Br, X0 @ W.Br, W.E, t0, max_dim=W.n)
    tau, bwd, dim = ek.trace_batch(W.V[idx], eps=eps, per_v=True)
    assert np.all(bwd <= eps), bwd.max()
    assert rel_err(tau, ref).max() <= 1e3 * eps, rel_err(tau, ref).max()
    if name == "c3":
        assert dim.max() <= W.n // 4, dim.max()
    ek.close()


def test_extended_krylov_capacity_is_flagged():
    """A basis capped below n cannot certify a tight target: LYAP_EPARTIAL, and with allow_partial the
    reported backward error is the last certified one (> eps), never a fabricated 0."""
    from paper_2312_08201_b200 import EKProblem, LyapError
    W = workloads.make("c1")
    X0 = scipy.linalg.solve_continuous_lyapunov(W.A0, -W.Q)
    t0 = float(np.sum(W.E * X0))
    ek = EKProblem(W.A0, W.Bl, W.Br, X0 @ W.Br, W.E, t0, max_dim=16)
    with pytest.raises(LyapError) as ei:
        ek.trace_batch(W.V[:8], eps=1e-12)
    assert ei.value.code == 6
    ek.close()
    ek = EKProblem(W.A0, W.Bl, W.Br, X0 @ W.Br, W.E, t0, max_dim=16)
    tau, dim, bwd = ek.trace_batch(W.V[:8], eps=1e-12, allow_partial=True)
    assert dim <= 16 and bwd > 1e-12 and np.all(np.isfinite(tau))
    ek.close()


# ----------------------------------------------------------------------------- NEXT row f4: stability filter
def _check_counts(P, A0, Bl, Br, V):
    got = P.unstable_count(V)
    for v, g in zip(V, got):
        ref = oracle.unstable_count(A0, Bl, Br, v)
        if g == -1:  # marginal: only allowed when the oracle's rightmost eigenvalue is at the axis
            assert abs(oracle.rightmost_real_part(A0, Bl, Br, v)) < 1e-8 * max(1.0, np.abs(A0).max()), v
        else:
            assert g == ref, (v, g, ref)
    return got


def test_stability_count_one_dof():
    """1-DOF: both eigenvalues cross at c = 2 a w + v phi^2 = 0 (oracle pin, closed form)."""
    w, a, phi = 1.3, 0.02, 0.7
    A0 = np.array([[0.0, w], [-w, -2 * a * w]])
    B = np.array([[0.0], [phi]])
    P = _problem(A0, B, B, np.eye(2), np.eye(2))
    vc = -2 * a * w / phi ** 2
    V = np.array([[-50.0], [-10.0], [vc * 3], [vc * 1.01], [vc * 0.99], [0.0], [0.3], [100.0]])
    got = _check_counts(P, A0, B, B, V)
    np.testing.assert_array_equal(got, [2, 2, 2, 2, 0, 0, 0, 0])
    P.close()


@pytest.mark.parametrize("n,k,seed", [(8, 1, 0), (20, 3, 1), (40, 2, 2)])
def test_stability_count_random(n, k, seed):
    """Random non-normal instances, v in [-20, 20]: unstable counts equal the oracle's eigenvalue counts."""
    rng = np.random.default_rng(300 + seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng)
    P = _problem(A0, Bl, Br, Q, E)
    V = rng.uniform(-20.0, 20.0, (60, k))
    got = _check_counts(P, A0, Bl, Br, V)
    assert (got == 0).any() and (got > 0).any()
    P.close()


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_stability_count_configs_negative_v(name):
    """Ex. 2/3-style negative parameters on the chain and the multi-agent network."""
    rng = np.random.default_rng(17)
    W = workloads.make(name)
    P = _problem(W.A0, W.Bl, W.Br, W.Q, W.E)
    lo, hi = (-5.0, 5.0) if name == "c3" else (-5.0, 5.0)
    V = rng.uniform(lo, hi, (40, W.k))
    got = _check_counts(P, W.A0, W.Bl, W.Br, V)
    assert (got == 0).any() and (got != 0).any()
    P.close()


def test_trace_batch_with_stability_filter():
    """opts.check_stable: unstable v come back as NaN with status LYAP_V_UNSTABLE (3) and are not
    solved; stable v match the oracle; the call is not LYAP_EPARTIAL."""
    rng = np.random.default_rng(23)
    A0, Bl, Br, Q, E = workloads.random_stable(16, 2, rng)
    V = rng.uniform(-15.0, 15.0, (50, 2))
    P = _problem(A0, Bl, Br, Q, E, check_stable=True)
    tau, st, ap, rs = P.trace_batch(V, return_diagnostics=True)
    stable = oracle.stable_mask(A0, Bl, Br, V)
    assert stable.any() and (~stable).any()
    np.testing.assert_array_equal(st == 3, ~stable)
    assert np.all(np.isnan(tau[~stable])) and np.all(ap[~stable] == 0)
    ref = oracle.trace_batch(A0, Bl, Br, Q, E, V[stable])
    assert rel_err(tau[stable], ref).max() <= RTOL
    P.close()


# ----------------------------------------------------------------------------- v-linear right-hand side
@pytest.mark.parametrize("n,k,seed", [(12, 2, 0), (30, 3, 1)])
def test_qlin_right_hand_side(n, k, seed):
    """lyap_setup_qlin: Q(v) = sum_i v_i Q_i (the projected equation of) solved as one
    capacitance system per v; traces and full X(v) against the oracle run with Q(v) formed explicitly."""
    rng = np.random.default_rng(70 + seed)
    A0, Bl, Br, _, E = workloads.random_stable(n, k, rng)
    Qs = []
    for _ in range(k):
        R = rng.standard_normal((n, 2))
        Qs.append(R @ R.T / n)
    Qs = np.array(Qs)
    V = rng.uniform(0.1, 2.0, (9, k))
    P = _problem(A0, Bl, Br, Qs, E)
    tau = P.trace_batch(V)
    X = P.solution(V[:3])
    for i, v in enumerate(V):
        Qv = np.tensordot(v, Qs, axes=1)
        ref, d = oracle.trace_EX(A0, Bl, Br, Qv, E, v, diagnostics=True)
        assert rel_err(tau[i], ref) <= RTOL, (i, tau[i], ref)
        if i < 3:
            assert np.abs(X[i] - d["X"]).max() <= 1e-9 * np.abs(d["X"]).max()
    P.close()


# ----------------------------------------------------------------------------- two-level preconditioner
@pytest.mark.parametrize("n,k,seed,p", [(30, 3, 0, 24), (64, 2, 1, 32), (13, 1, 2, 8)])
def test_two_level_preconditioner_random(n, k, seed, p):
    """opts.coarse: the two-level preconditioner (coarse space from the off-block TSVD, exact Galerkin
    coarse solve per v) changes the Krylov path, not the answer: traces vs the oracle, every v."""
    rng = np.random.default_rng(90 + seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng)
    V = rng.uniform(0.05, 3.0, (29, k))
    V[3, 0] = 0.0  # a masked column
    P = _problem(A0, Bl, Br, Q, E, coarse=p, batch=8)
    tau, st, ap, rs = P.trace_batch(V, return_diagnostics=True)
    assert np.all(st == 0), (st, rs)
    assert np.all(rs <= 1e-12)
    assert rel_err(tau, oracle.trace_batch(A0, Bl, Br, Q, E, V)).max() <= RTOL
    P.close()


@pytest.mark.parametrize("name,p", [("c1", 64), ("c2", 128)])
def test_two_level_preconditioner_configs(name, p):
    """c1 / c2 with the two-level preconditioner: oracle goldens, and fewer T-applications than the
    pair blocks alone (measured: c2 high corner 95 -> 68 GMRES iterations at p = 128)."""
    W = workloads.make(name)
    g = _golden(name)
    idx = np.array(g["indices"])
    P0 = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, coarse=0)
    P0.trace_batch(W.V)
    P1 = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, coarse=p)
    tau, st, ap, rs = P1.trace_batch(W.V, return_diagnostics=True)
    a0 = P0.stats["k1_vectors"]
    P1.reset_stats()
    P1.trace_batch(W.V)
    a1 = P1.stats["k1_vectors"]
    assert np.all(st == 0)
    assert rel_err(tau[idx], np.array(g["traces"])).max() <= RTOL
    assert a1 < a0, (a0, a1)
    P0.close()
    P1.close()


# ----------------------------------------------------------------------------- mixed precision
@pytest.mark.parametrize("n,k,seed", [(30, 3, 0), (64, 2, 1), (13, 1, 2), (40, 4, 3),
                                      # npad a multiple of 128: the tcgen05 path (fused epilogue for
                                      # k = 1, 2, 4; k1_epi for k = 3), real eigenvalues included
                                      (150, 2, 4), (200, 4, 5), (130, 1, 6), (140, 3, 7),
                                      # npad = 256 / 384: the 3xFP16 tcgen05 path (k = 3 unfused)
                                      (250, 3, 8), (380, 2, 9)])
def test_mixed_precision_random(n, k, seed):
    """opts.mixed = 1: Krylov steps with the 3xTF32 T-apply, every cycle restarted from
    the exact FP64 true residual.  The stopping test is the FP64 one, so every v meets tol = 1e-12 and
    the traces match the oracle; only the VERIFY applications are exact."""
    rng = np.random.default_rng(120 + seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng)
    V = rng.uniform(0.05, 3.0, (29, k))
    V[3, 0] = 0.0  # a masked column
    P = _problem(A0, Bl, Br, Q, E, mixed=1, batch=8)
    tau, st, ap, rs = P.trace_batch(V, return_diagnostics=True)
    assert np.all(st == 0), (st, rs)
    assert np.all(rs <= 1e-12)
    assert rel_err(tau, oracle.trace_batch(A0, Bl, Br, Q, E, V)).max() <= RTOL
    s = P.stats
    assert 0 < s["k1_exact_vectors"] < s["k1_vectors"], s
    P.close()


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_mixed_precision_configs(name):
    """mixed = 1 forced on the small configurations (auto turns it on only for n > 1536): oracle
    goldens at 1e-9, and the mixed and FP64-only engines agree to the solver tolerance."""
    W = workloads.make(name)
    g = _golden(name)
    idx = np.array(g["indices"])
    P1 = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, mixed=1)
    tau1, st, ap, rs = P1.trace_batch(W.V, return_diagnostics=True)
    assert np.all(st == 0)
    assert np.all(rs <= 1e-12)
    assert rel_err(tau1[idx], np.array(g["traces"])).max() <= RTOL
    exact = P1.stats["k1_exact_vectors"]
    assert exact < 0.5 * P1.stats["k1_vectors"]
    P0 = _problem(W.A0, W.Bl, W.Br, W.Q, W.E, mixed=0)
    tau0 = P0.trace_batch(W.V)
    assert P0.stats["k1_exact_vectors"] == P0.stats["k1_vectors"]
    assert rel_err(tau1, tau0).max() <= 1e-10
    P0.close()
    P1.close()


@pytest.mark.parametrize("n,k,seed", [(200, 4, 0), (256, 2, 1), (150, 3, 2), (1700, 4, 3), (250, 3, 4)])
def test_k1_mixed_apply_against_paper_blocks(n, k, seed):
    """The mixed-precision operator (lyap_apply_C_mixed: the Cauchy part on the tcgen05 3xTF32 GEMM,
    T_d and sigma o X in FP64) against the same entrywise operator of eqs. (N1M1)/(N2M1)/(N1M2):
    within the 3xTF32 accuracy (1e-4 of the largest entry), and visibly NOT exact -- the FP64
    apply_C of the same vectors is within 1e-12 (the refinement's residual check needs that one)."""
    import torch
    rng = np.random.default_rng(40 + seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng)
    P = _problem(A0, Bl, Br, Q, E, mixed=1)
    st = P.export_state()
    npairs, npad = st["n_pairs"], st["npad"]
    lam, br, bl = _complex_factors(st, n)
    L = 1.0 / (lam[:, None] + lam[None, :])
    F = np.einsum("ij,is,it->jst", L, br, bl)
    nvec = 7
    sig = rng.uniform(-2, 3, (nvec, k))
    Gs = [_unfold(_fold(rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)), npairs, npad), npairs, n)
          for _ in range(nvec)]
    Xt = torch.tensor(np.stack([_fold(G, npairs, npad) for G in Gs]), device="cuda")
    St = torch.tensor(sig, device="cuda")
    Ym = P.apply_C(Xt, St, mixed=True).cpu().numpy()
    Y64 = P.apply_C(Xt, St).cpu().numpy()
    worst = 0.0
    for v in range(nvec):
        G = Gs[v]
        TG = np.einsum("jst,tj->sj", F, G) + np.einsum("jt,ij,is,ti->sj", bl, L, br, G)
        expect = _fold(sig[v][:, None] * G - TG, npairs, npad)
        scale = np.abs(expect).max()
        np.testing.assert_allclose(Y64[v], expect, rtol=0, atol=1e-12 * scale)
        err = np.abs(Ym[v] - expect).max() / scale
        worst = max(worst, err)
        assert err <= 1e-4, err
        assert np.all(Ym[v][:, n:] == 0.0)
    assert worst > 1e-12  # the inexact operator really is the float one
    P.close()
