"""CPU pin of the mathematics the CUDA path implements, written
independently of the CUDA code in plain complex NumPy: the symmetric nk capacitance system
(Delta(v) - T) g = g0, trace = t0 + 2 sum G o H^T, must reproduce the oracle's Bartels-Stewart traces
(the paper's SMW route, restricted to symmetric solutions); and the real pair
folding of the Cauchy coupling must equal the complex sum it replaces."""
import numpy as np
import pytest

import oracle
import workloads


def nk_form_traces(A0, Bl, Br, Q, E, V):
    lam, S = np.linalg.eig(A0)
    Si = np.linalg.inv(S)
    n, k = Bl.shape
    L = 1.0 / (lam[:, None] + lam[None, :])
    bl, br = Si @ Bl, S.T @ Br
    X0t = -L * (Si @ Q @ Si.T)
    Et = S.T @ (0.5 * (E + E.T)) @ S
    g0 = (br.T @ X0t).ravel()  # G0 = B^r^T X~0, k x n, row-major (t, j)
    H = (Et * L) @ bl
    t0 = np.sum(Et * X0t)
    # T as an explicit nk x nk matrix, entrywise from eqs. (N1M1) and (N2M1)/(N1M2)
    F = np.einsum("ij,is,it->jst", L, br, bl)
    T = np.zeros((k * n, k * n), complex)
    for s in range(k):
        for t in range(k):
            T[s * n:(s + 1) * n, t * n:(t + 1) * n] += np.diag(F[:, s, t])
            T[s * n:(s + 1) * n, t * n:(t + 1) * n] += (bl[:, t][:, None] * L.T) * br[:, s][None, :]
    out = []
    for v in V:
        Dinv = np.repeat(1.0 / np.asarray(v, float), n)
        g = np.linalg.solve(np.diag(Dinv) - T, g0).reshape(k, n)
        out.append((t0 + 2.0 * np.sum(g * H.T)).real)
    return np.array(out)


@pytest.mark.parametrize("n,k,seed,same_b", [(5, 1, 0, True), (9, 2, 1, False), (12, 3, 2, False),
                                             (17, 4, 3, True), (26, 2, 4, False)])
def test_nk_capacitance_form_equals_oracle(n, k, seed, same_b):
    rng = np.random.default_rng(200 + seed)
    A0, Bl, Br, Q, E = workloads.random_stable(n, k, rng, same_b=same_b)
    V = rng.uniform(0.05, 2.0, (6, k))
    ref = oracle.trace_batch(A0, Bl, Br, Q, E, V)
    got = nk_form_traces(A0, Bl, Br, Q, E, V)
    np.testing.assert_allclose(got, ref, rtol=1e-9)


def test_nk_form_on_c1_corners():
    W = workloads.make("c1")
    idx = W.corner_indices()
    ref = oracle.trace_batch(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[idx])
    np.testing.assert_allclose(nk_form_traces(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[idx]), ref, rtol=1e-9)


def test_pair_folding_of_the_cauchy_coupling():
    """For a conjugate pair (i, i~) and output index j: L_ij R + L_i~j conj(R) = [[a+c, d-b], [b+d, a-c]] [x; y]
    with a+ib = L_ij, c+id = L_i~j, R = x+iy; and the mixed real/pair variants."""
    rng = np.random.default_rng(7)
    for _ in range(100):
        li = complex(-rng.uniform(0.01, 2), rng.uniform(0.1, 5))
        lj = complex(-rng.uniform(0.01, 2), rng.uniform(-5, 5))
        R = complex(*rng.standard_normal(2))
        L1, L2 = 1 / (li + lj), 1 / (np.conj(li) + lj)
        a, b, c, d = L1.real, L1.imag, L2.real, L2.imag
        z = L1 * R + L2 * np.conj(R)
        M = np.array([[a + c, d - b], [b + d, a - c]])
        np.testing.assert_allclose(M @ [R.real, R.imag], [z.real, z.imag], rtol=1e-13, atol=1e-13)
        # real output j (lambda_j real): the sum is real and equals [2a, -2b] . [x, y]
        ljr = -rng.uniform(0.01, 2)
        L1r = 1 / (li + ljr)
        zr = L1r * R + np.conj(L1r) * np.conj(R)
        assert abs(zr.imag) < 1e-12
        assert zr.real == pytest.approx(2 * L1r.real * R.real - 2 * L1r.imag * R.imag, rel=1e-13, abs=1e-13)
