"""Exploration (not product code, not the oracle): tile-shared projection for the nk capacitance
system C(v) g = g0, C(v) = Delta(v) - T, in torch complex128 (CPU or GPU).

A tile = B neighbouring grid points.  They share one search space Z (orthonormal, N = nk rows) and
T Z (every T-application is reused by every member: C(v) Z = Delta(v) Z - T Z).  Greedy: each step
adds P(v)^{-1} r(v) of the p worst members (block CGS2), applies T to the new columns, and every
unconverged member re-solves its projected system (Galerkin or minimal residual via the normal
equations plus one refinement), with explicit residuals.  Prints T-applies per v and the final dim.

python tools/explore/tile_galerkin.py c2 8x8 [p] [galerkin|minres] [device]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import workloads  # noqa: E402


class Sys:
    def __init__(self, W, dev):
        t = time.time()
        lam, S = np.linalg.eig(W.A0)
        S_t = torch.tensor(S, device=dev)
        Si = torch.linalg.inv(S_t)
        lam_t = torch.tensor(lam, device=dev)
        self.lam_np = lam
        self.k, self.n, self.dev = W.k, W.n, dev
        self.L = 1.0 / (lam_t[:, None] + lam_t[None, :])
        Bl = torch.tensor(W.Bl, device=dev, dtype=torch.complex128)
        Br = torch.tensor(W.Br, device=dev, dtype=torch.complex128)
        self.bl = Si @ Bl
        self.br = S_t.T @ Br
        Q = torch.tensor(W.Q, device=dev, dtype=torch.complex128)
        E = torch.tensor(0.5 * (W.E + W.E.T), device=dev, dtype=torch.complex128)
        X0 = -self.L * (Si @ Q @ Si.T)
        Et = S_t.T @ E @ S_t
        self.g0 = (self.br.T @ X0)  # k x n
        self.H = (Et * self.L) @ self.bl  # n x k
        self.t0 = torch.sum(Et * X0).real.item()
        self.F = torch.einsum("ij,is,it->jst", self.L, self.br, self.bl)  # n x k x k
        self.LT = self.L.T.contiguous()
        self.applies = 0
        print(f"setup {time.time() - t:.1f}s", flush=True)

    def T(self, G):  # G: p x k x n -> p x k x n
        p = G.shape[0]
        self.applies += p
        R = (self.br[:, None, :, None] * G.permute(2, 0, 1)[:, :, None, :]).reshape(self.n, -1)  # i,(b,s,t)
        U = (self.LT @ R).reshape(self.n, p, self.k, self.k)
        Y = torch.einsum("jst,btj->bsj", self.F, G) + torch.einsum("jt,jbst->bsj", self.bl, U)
        return Y

    def minv(self, V):  # V: B x k -> B x n x k x k
        sig = 1.0 / V
        M = torch.diag_embed(sig.to(torch.complex128))[:, None, :, :] - self.F[None]
        return torch.linalg.inv(M)

    def pairs(self):
        """(nrep, 2) eigen indices [j, conj partner] (chains: all eigenvalues complex)."""
        if hasattr(self, "_idx"):
            return self._idx
        lam = self.lam_np
        n = len(lam)
        partner = -np.ones(n, int)
        for j in range(n):
            if partner[j] >= 0:
                continue
            d = np.abs(lam - np.conj(lam[j]))
            d[j] = np.inf
            p = int(np.argmin(d))
            assert partner[p] < 0 and abs(lam[j].imag) > 0
            partner[j], partner[p] = p, j
        reps = [(j, partner[j]) for j in range(n) if partner[j] > j]
        self._idx = torch.tensor(reps, device=self.dev)
        return self._idx

    def pminv(self, V):
        """Pair-block preconditioner: exact diagonal blocks of C(v) over the unknowns of one conjugate
        pair {j, conj j} (T_d plus the T_o self-coupling L[conj j, j] = 1/(2 Re lambda_j)).
        Returns (nrep x 2k x 2k) inverse per v: B x nrep x 2k x 2k, ordering (s, a)."""
        idx = self.pairs()
        k = self.k
        nr = idx.shape[0]
        Lsub = self.L[idx[:, None, :], idx[:, :, None]]  # [r, a, b] = L[idx_b, idx_a]
        bl = self.bl[idx]  # r, a, t
        br = self.br[idx]  # r, b, s
        To = torch.einsum("rat,rab,rbs->rsatb", bl, Lsub, br)
        Fd = self.F[idx]  # r, a, s, t
        eye2 = torch.eye(2, dtype=torch.complex128, device=self.dev)
        Td = torch.einsum("rast,ab->rsatb", Fd, eye2)
        base = -(To + Td).reshape(nr, 2 * k, 2 * k)
        sig = (1.0 / V).to(torch.complex128)  # B x k
        D = torch.diag_embed(sig.repeat_interleave(2, dim=1))  # B x 2k x 2k, (s, a) order
        return torch.linalg.inv(base[None] + D[:, None])

    def papply(self, Pm, R):  # Pm: B x nrep x 2k x 2k, R: B x k x n
        idx = self.pairs()
        B = R.shape[0]
        r = R[:, :, idx]  # B, k, nrep, 2
        r = r.permute(0, 2, 1, 3).reshape(B, -1, 2 * self.k, 1)
        z = (Pm @ r)[..., 0].reshape(B, -1, self.k, 2).permute(0, 2, 1, 3)
        Z = torch.zeros_like(R)
        Z[:, :, idx] = z
        return Z

    def trace(self, G):  # G: B x k x n
        return self.t0 + 2 * torch.einsum("bsj,js->b", G, self.H).real


def tile_solve(sm, V, p=4, mode="galerkin", tol=1e-12, maxr=6000, verbose=False, prec="pair"):
    dev = sm.dev
    k, n = sm.k, sm.n
    N = k * n
    B = V.shape[0]
    Vt = torch.tensor(V, device=dev)
    sig = (1.0 / Vt).to(torch.complex128)  # B x k
    sigN = sig.repeat_interleave(n, dim=1)  # B x N
    g0 = sm.g0.reshape(N)
    bn = torch.linalg.norm(g0)
    Minv = sm.minv(Vt) if prec == "td" else sm.pminv(Vt)
    Z = torch.zeros(N, 0, dtype=torch.complex128, device=dev)
    TZ = torch.zeros(N, 0, dtype=torch.complex128, device=dev)
    R = g0[None, :].repeat(B, 1)
    res = torch.ones(B, dtype=torch.float64, device=dev)
    Y = None
    a0 = sm.applies
    steps = 0
    t_small = 0.0
    hybrid = mode.startswith("hybrid")
    grow = float(mode.split(":")[1]) if ":" in mode else 1.3
    next_check = 0
    dirs = {}  # hybrid: member -> (its last direction, T of it)
    nsolves = 0
    while res.max() > tol and Z.shape[1] < maxr:
        steps += 1
        act = torch.nonzero(res > tol).flatten()
        if hybrid and Z.shape[1] > 0 and Z.shape[1] < next_check and all(int(b) in dirs for b in act):
            # block-Krylov continuation: z_b = P_b^{-1} C(v_b) d_b with T d_b already known
            order = act
            Rp = torch.stack([sigN[b] * dirs[int(b)][0] - dirs[int(b)][1] for b in act]).reshape(-1, k, n)
        else:
            order = act[torch.argsort(-res[act])][:p]
            Rp = R[order].reshape(-1, k, n)
        if prec == "td":
            D = torch.einsum("bjst,btj->bsj", Minv[order], Rp).reshape(-1, N).T  # N x p
        else:
            D = sm.papply(Minv[order], Rp).reshape(-1, N).T
        for _ in range(2):
            D = D - Z @ (Z.conj().T @ D)
        Qd, Rd = torch.linalg.qr(D)
        keep = torch.abs(torch.diagonal(Rd)) > 1e-13 * torch.abs(torch.diagonal(Rd)).max()
        Qd = Qd[:, keep]
        if Qd.shape[1] == 0:
            break
        TQ = sm.T(Qd.T.reshape(-1, k, n)).reshape(-1, N).T
        Z = torch.cat([Z, Qd], 1)
        TZ = torch.cat([TZ, TQ], 1)
        if hybrid:
            dirs = {}
            kept = [int(b) for b, kp in zip(order, keep) if kp]
            for i, b in enumerate(kept):
                dirs[b] = (Qd[:, i], TQ[:, i])
            if Z.shape[1] < next_check and all(int(b) in dirs for b in act):
                continue  # no solve this step
            next_check = max(int(grow * Z.shape[1]), Z.shape[1] + len(act))
        nsolves += 1
        # projected solves for the unconverged members
        ts = time.time()
        r = Z.shape[1]
        CZ_parts = None
        if mode == "galerkin":
            Phi = [Z[t * n:(t + 1) * n].conj().T @ Z[t * n:(t + 1) * n] for t in range(k)]
            Psi = Z.conj().T @ TZ
            M = -Psi[None].repeat(len(act), 1, 1)
            for t in range(k):
                M = M + sig[act, t][:, None, None] * Phi[t][None]
            rhs = (Z.conj().T @ g0)[None, :, None].repeat(len(act), 1, 1)
            Ya = torch.linalg.solve(M, rhs)[..., 0]  # a x r
        else:  # minimal residual via normal equations + one refinement
            G1 = [Z[t * n:(t + 1) * n].conj().T @ Z[t * n:(t + 1) * n] for t in range(k)]
            G2 = [Z[t * n:(t + 1) * n].conj().T @ TZ[t * n:(t + 1) * n] for t in range(k)]
            G3 = TZ.conj().T @ TZ
            NE = G3[None].repeat(len(act), 1, 1).clone()
            for t in range(k):
                s = sig[act, t].real
                NE = NE + (s ** 2)[:, None, None] * G1[t][None] - s[:, None, None] * (G2[t] + G2[t].conj().T)[None]
            def cz_h(Rv):  # (Delta Z - TZ)^H r for each member: a x r
                out = -(TZ.conj().T @ Rv.T).T
                for t in range(k):
                    out = out + sig[act, t].real[:, None] * (Z[t * n:(t + 1) * n].conj().T @ Rv[:, t * n:(t + 1) * n].T).T
                return out
            Ya = torch.linalg.solve(NE, cz_h(g0[None].repeat(len(act), 1))[..., None])[..., 0]
            for _ in range(2):
                Ra = g0[None] - sigN[act] * (Z @ Ya.T).T + (TZ @ Ya.T).T
                Ya = Ya + torch.linalg.solve(NE, cz_h(Ra)[..., None])[..., 0]
        if dev != "cpu":
            torch.cuda.synchronize()
        t_small += time.time() - ts
        Ra = g0[None] - sigN[act] * (Z @ Ya.T).T + (TZ @ Ya.T).T
        R[act] = Ra
        res[act] = torch.linalg.norm(Ra, dim=1) / bn
        if verbose and steps % 10 == 0:
            print(f"   step {steps} dim {r} worst {res.max().item():.2e} active {int((res > tol).sum())}", flush=True)
    if verbose:
        print(f"   solves {nsolves}", flush=True)
    return sm.applies - a0, Z.shape[1], steps, t_small


def gmres(sm, v, prec="pair", tol=1e-12, m=1000):
    """Right-preconditioned GMRES (CGS2, no restart) for one v: T-applies to convergence."""
    dev = sm.dev
    k, n = sm.k, sm.n
    Vt = torch.tensor(v[None], device=dev)
    Pm = sm.minv(Vt) if prec == "td" else sm.pminv(Vt)
    ap = (lambda R: torch.einsum("bjst,btj->bsj", Pm, R)) if prec == "td" else (lambda R: sm.papply(Pm, R))
    sig = (1.0 / Vt).to(torch.complex128).repeat_interleave(n, dim=1)[0]
    g0 = sm.g0.reshape(-1)
    beta = torch.linalg.norm(g0)
    Qb = [g0 / beta]
    H = torch.zeros(m + 1, m, dtype=torch.complex128, device=dev)
    for j in range(m):
        z = ap(Qb[j].reshape(1, k, n))
        w = (sig * z.reshape(-1) - sm.T(z).reshape(-1))
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
    tshape = tuple(int(x) for x in sys.argv[2].split("x"))
    p = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    mode = sys.argv[4] if len(sys.argv) > 4 else "galerkin"
    dev = sys.argv[5] if len(sys.argv) > 5 else "cpu"
    which = sys.argv[6].split(",") if len(sys.argv) > 6 else ["low", "mid", "high", "mixed"]
    prec = sys.argv[7] if len(sys.argv) > 7 else "pair"
    W = workloads.make(name)
    sm = Sys(W, dev)
    shp = W.grid_shape
    if mode == "gmres":
        pts = {"low": [0] * len(shp), "high": [s - 1 for s in shp], "mid": [s // 2 for s in shp],
               "mixed": [s - 1 if i == 0 else 0 for i, s in enumerate(shp)], "p80": [int(0.8 * s) for s in shp]}
        for label in which:
            v = W.V[int(np.ravel_multi_index(tuple(pts[label]), shp))]
            t = time.time()
            out = [f"{pr}:{gmres(sm, v, prec=pr)}" for pr in ("td", "pair")]
            print(f"{name} gmres {label} v={np.round(v, 3)}: " + " ".join(out) + f" ({time.time() - t:.1f}s)", flush=True)
        return
    starts = {"low": [0] * len(shp), "mid": [s // 2 - t // 2 for s, t in zip(shp, tshape)],
              "high": [s - t for s, t in zip(shp, tshape)],
              "mixed": [s - t if i == 0 else 0 for i, (s, t) in enumerate(zip(shp, tshape))]}
    for label in which:
        start = starts[label]
        idx = [int(np.ravel_multi_index(tuple(st + o for st, o in zip(start, off)), shp)) for off in np.ndindex(*tshape)]
        t = time.time()
        a, r, st, ts = tile_solve(sm, W.V[idx], p=p, mode=mode, verbose=True, prec=prec)
        print(f"{name} {mode} {prec} p={p} tile {label} {tshape}: {a} T-applies / {len(idx)} v = {a / len(idx):.2f}/v, "
              f"dim {r}, steps {st}, small-solve {ts:.1f}s, total {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
