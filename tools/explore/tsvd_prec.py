"""Exploration (not product code): GMRES iterations with the paper's TSVD preconditioner (eq. (prec),
PAPER.md:414-457, p-bar > 0) on top of the pair-block diagonal part.  Complex unfolded torch.

P(v) = M(v) - U S V^H,  M(v) = Delta(v) - T_d - T_o|pair (pair-block diagonal, exact per v),
U S V^H = rank-p TSVD of T_o - T_o|pair (randomized range finder with power iterations, computed
once); P^{-1} by Sherman-Morrison-Woodbury with the p x p capacitance S^{-1} - V^H M^{-1} U per v.

python tools/explore/tsvd_prec.py c5 50,100,200 [device]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/", 1)[0])
import workloads  # noqa: E402
from tile_galerkin import Sys  # noqa: E402


def to_apply(sm, G, adjoint=False):
    """T_o G (dense Cauchy coupling) minus its pair-block part; G: p x k x n."""
    k, n = sm.k, sm.n
    p = G.shape[0]
    idx = sm.pairs()
    if not adjoint:
        R = (sm.br[:, None, :, None] * G.permute(2, 0, 1)[:, :, None, :]).reshape(n, -1)
        U = (sm.LT @ R).reshape(n, p, k, k)
        Y = torch.einsum("jt,jbst->bsj", sm.bl, U)
    else:
        Wm = (sm.bl.conj()[:, None, None, :] * G.permute(2, 0, 1)[:, :, :, None]).reshape(n, -1)  # j,(b,s,t)
        Rm = (sm.L.conj() @ Wm).reshape(n, p, k, k)  # i, b, s, t
        Y = torch.einsum("is,ibst->bti", sm.br.conj(), Rm)
    a, b = idx[:, 0], idx[:, 1]
    Yp = torch.zeros_like(Y)
    for (jj, ii) in ((a, a), (a, b), (b, a), (b, b)):
        if not adjoint:  # out_{s,j} += sum_t bl_jt L_ij br_is G_ti
            c = sm.L[ii, jj][None, None, :]
            term = torch.einsum("jt,js,btj->bsj", sm.bl[jj], sm.br[ii], G[:, :, ii]) * c
            Yp[:, :, jj] += term
        else:  # out_{t,i} += sum_s conj(bl_jt L_ij br_is) G_sj
            c = sm.L[ii, jj].conj()[None, None, :]
            term = torch.einsum("jt,js,bsj->btj", sm.bl[jj].conj(), sm.br[ii].conj(), G[:, :, jj]) * c
            Yp[:, :, ii] += term
    return Y - Yp


def rsvd(sm, p, q=2, over=20):
    k, n = sm.k, sm.n
    g = torch.Generator(device=sm.dev).manual_seed(0)
    l = p + over
    Om = torch.randn(l, k, n, generator=g, device=sm.dev, dtype=torch.float64).to(torch.complex128)
    Y = to_apply(sm, Om)
    for _ in range(q):
        Qm, _ = torch.linalg.qr(Y.reshape(l, -1).T)
        Z = to_apply(sm, Qm.T.reshape(l, k, n), adjoint=True)
        Qz, _ = torch.linalg.qr(Z.reshape(l, -1).T)
        Y = to_apply(sm, Qz.T.reshape(l, k, n))
    Qm, _ = torch.linalg.qr(Y.reshape(l, -1).T)  # N x l
    TH = to_apply(sm, Qm.T.reshape(l, k, n), adjoint=True).reshape(l, -1)  # row i = (T^H q_i)^T
    B = TH.conj()  # B = Q^H T  (l x N)
    Ub, S, Vh = torch.linalg.svd(B, full_matrices=False)
    U = Qm @ Ub[:, :p]
    return U, S[:p], Vh[:p].conj().T  # T ~ U diag(S) V^H


def gmres_prec(sm, v, pinv, tol=1e-12, m=1000):
    k, n = sm.k, sm.n
    dev = sm.dev
    Vt = torch.tensor(v[None], device=dev)
    sig = (1.0 / Vt).to(torch.complex128).repeat_interleave(n, dim=1)[0]
    g0 = sm.g0.reshape(-1)
    beta = torch.linalg.norm(g0)
    Qb = [g0 / beta]
    H = torch.zeros(m + 1, m, dtype=torch.complex128, device=dev)
    for j in range(m):
        z = pinv(Qb[j])
        w = sig * z - sm.T(z.reshape(1, k, n)).reshape(-1)
        Qm = torch.stack(Qb, 1)
        for _ in range(2):
            h = Qm.conj().T @ w
            H[: j + 1, j] += h
            w = w - Qm @ h
        H[j + 1, j] = torch.linalg.norm(w)
        Qb.append(w / H[j + 1, j])
        e = torch.zeros(j + 2, dtype=torch.complex128, device=dev)
        e[0] = beta
        y = torch.linalg.lstsq(H[: j + 2, : j + 1], e[:, None]).solution[:, 0]
        if torch.linalg.norm(H[: j + 2, : j + 1] @ y - e) <= 0.5 * tol * beta:
            return j + 1
    return m


def main():
    name = sys.argv[1]
    ps = [int(x) for x in sys.argv[2].split(",")]
    dev = sys.argv[3] if len(sys.argv) > 3 else "cuda"
    W = workloads.make(name)
    sm = Sys(W, dev)
    k, n = sm.k, sm.n
    shp = W.grid_shape
    pts = {"high": [s - 1 for s in shp], "p80": [int(0.8 * s) for s in shp], "mid": [s // 2 for s in shp],
           "mixed": [s - 1 if i == 0 else 0 for i, s in enumerate(shp)], "p65": [int(0.65 * s) for s in shp]}
    t = time.time()
    pmax = max(ps)
    U, S, V = rsvd(sm, pmax)
    # check the TSVD: ||T_o' x - U S V^H x|| / ||T_o' x|| on a random x
    x = torch.randn(1, k, n, device=dev, dtype=torch.float64).to(torch.complex128)
    tx = to_apply(sm, x).reshape(-1)
    ax = U @ (S.to(torch.complex128) * (V.conj().T @ x.reshape(-1)))
    print(f"rsvd p={pmax}: {time.time() - t:.1f}s; sigma_1 {S[0].item():.3e} sigma_p {S[-1].item():.3e}; "
          f"rel err on random x {torch.linalg.norm(tx - ax).item() / torch.linalg.norm(tx).item():.3e}", flush=True)
    for label, pt in pts.items():
        v = W.V[int(np.ravel_multi_index(tuple(pt), shp))]
        Vt = torch.tensor(v[None], device=dev)
        Pm = sm.pminv(Vt)
        minv = lambda r: sm.papply(Pm, r.reshape(1, k, n)).reshape(-1)
        out = [f"pair:{gmres_prec(sm, v, minv)}"]
        sig = (1.0 / Vt).to(torch.complex128).repeat_interleave(n, dim=1)[0]
        for p in ps:
            # two-level (coarse-grid) preconditioner with a v-independent space Z: per v only the
            # p x p Galerkin matrix E(v) = Z^H C(v) Z (cheap from Gram blocks) is factored
            for zname, Z in (("V", V[:, :p]), ("UV", torch.linalg.qr(torch.cat([U[:, : p // 2], V[:, : p // 2]], 1))[0])):
                TZ = sm.T(Z.T.reshape(-1, k, n)).reshape(-1, n * k).T
                CZ = sig[:, None] * Z - TZ
                Einv = torch.linalg.inv(Z.conj().T @ CZ)

                def pinv2(r, Z=Z, CZ=CZ, Einv=Einv):
                    w = Einv @ (Z.conj().T @ r)
                    return Z @ w + minv(r - CZ @ w)
                out.append(f"2L{zname}{p}:{gmres_prec(sm, v, pinv2)}")
        for p in ps:
            Up, Sp, Vp = U[:, :p], S[:p], V[:, :p]
            MU = torch.stack([minv(Up[:, i]) for i in range(p)], 1)  # N x p
            K = torch.diag(1.0 / Sp.to(torch.complex128)) - Vp.conj().T @ MU
            Kinv = torch.linalg.inv(K)

            def pinv(r, MU=MU, Kinv=Kinv, Vp=Vp):
                z = minv(r)
                return z + MU @ (Kinv @ (Vp.conj().T @ z))
            out.append(f"p{p}:{gmres_prec(sm, v, pinv)}")
        print(f"{name} {label} v={np.round(v, 3)}: " + " ".join(out), flush=True)


if __name__ == "__main__":
    main()
