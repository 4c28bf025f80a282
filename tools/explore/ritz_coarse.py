"""Exploration: two-level preconditioner with a coarse space of harmonic Ritz vectors collected from
GMRES solves at seed parameter vectors (the recycling idea of PAPER.md:380-391 used as a coarse
space), against the TSVD right singular space.  python tools/explore/ritz_coarse.py c5 [s] [device]"""
import itertools
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/", 1)[0])
import workloads  # noqa: E402
from tile_galerkin import Sys  # noqa: E402
from tsvd_prec import gmres_prec, rsvd  # noqa: E402


def gmres_ritz(sm, v, s, tol=1e-12, m=600):
    """Right-preconditioned GMRES; returns the s harmonic Ritz vectors of smallest magnitude (x-space
    search directions Z y) of the final Arnoldi relation."""
    k, n = sm.k, sm.n
    dev = sm.dev
    Vt = torch.tensor(v[None], device=dev)
    Pm = sm.pminv(Vt)
    minv = lambda r: sm.papply(Pm, r.reshape(1, k, n)).reshape(-1)
    sig = (1.0 / Vt).to(torch.complex128).repeat_interleave(n, dim=1)[0]
    g0 = sm.g0.reshape(-1)
    beta = torch.linalg.norm(g0)
    Qb, Zs = [g0 / beta], []
    H = torch.zeros(m + 1, m, dtype=torch.complex128, device=dev)
    for j in range(m):
        z = minv(Qb[j])
        Zs.append(z)
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
            break
    mm = j + 1
    Hm = H[: mm + 1, :mm]
    # harmonic Ritz: (Hm^H Hm) p = theta Hm[:mm]^H p  -> smallest |theta|
    import scipy.linalg
    A = (Hm.conj().T @ Hm).resolve_conj().cpu().numpy()
    B = Hm[:mm, :mm].conj().T.resolve_conj().cpu().numpy()
    th, P = scipy.linalg.eig(A, B)
    order = np.argsort(np.abs(th))[:s]
    Pt = torch.tensor(P[:, order], device=dev)
    return torch.stack(Zs, 1) @ Pt, mm


def main():
    name = sys.argv[1]
    s = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dev = sys.argv[3] if len(sys.argv) > 3 else "cuda"
    W = workloads.make(name)
    sm = Sys(W, dev)
    k, n = sm.k, sm.n
    lo, hi = W.V.min(0), W.V.max(0)
    seeds = [np.array([hi[t] if b else lo[t] for t, b in enumerate(bits)]) for bits in itertools.product((0, 1), repeat=k)]
    cols = []
    for v in seeds:
        U, mm = gmres_ritz(sm, v, s)
        cols.append(U)
        print("seed", np.round(v, 3), "its", mm, flush=True)
    Zr, _ = torch.linalg.qr(torch.cat(cols, 1))
    Ut, St, Vt_ = rsvd(sm, 128)
    shp = W.grid_shape
    pts = {"high": [x - 1 for x in shp], "p80": [int(0.8 * x) for x in shp], "mid": [x // 2 for x in shp],
           "mixed": [x - 1 if i == 0 else 0 for i, x in enumerate(shp)], "p65": [int(0.65 * x) for x in shp]}
    for label, pt in pts.items():
        v = W.V[int(np.ravel_multi_index(tuple(pt), shp))]
        Vv = torch.tensor(v[None], device=dev)
        Pm = sm.pminv(Vv)
        minv = lambda r: sm.papply(Pm, r.reshape(1, k, n)).reshape(-1)
        sig = (1.0 / Vv).to(torch.complex128).repeat_interleave(n, dim=1)[0]
        out = [f"pair:{gmres_prec(sm, v, minv)}"]
        for zname, Z in (("ritz", Zr), ("tsvd128", Vt_[:, :128]),
                         ("both", torch.linalg.qr(torch.cat([Zr, Vt_[:, :64]], 1))[0])):
            TZ = sm.T(Z.T.reshape(-1, k, n)).reshape(-1, n * k).T
            CZ = sig[:, None] * Z - TZ
            Einv = torch.linalg.inv(Z.conj().T @ CZ)

            def pinv2(r, Z=Z, CZ=CZ, Einv=Einv):
                w = Einv @ (Z.conj().T @ r)
                return Z @ w + minv(r - CZ @ w)
            out.append(f"{zname}({Z.shape[1]}):{gmres_prec(sm, v, pinv2)}")
        print(f"{name} {label}: " + " ".join(out), flush=True)


if __name__ == "__main__":
    main()
