"""CPU exploration (not product code, not the oracle): iteration counts of Krylov strategies for the
nk capacitance system C(v) g = g0, complex unfolded NumPy.  Used to choose the GPU
solver design; prints T-applications per v for each strategy on sample grid points.

python tools/explore/krylov_strategies.py c2 [strategies...]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import workloads  # noqa: E402


class Sys:
    def __init__(self, W):
        lam, S = np.linalg.eig(W.A0)
        Si = np.linalg.inv(S)
        self.k, self.n = W.k, W.n
        self.lam = lam
        self.L = 1.0 / (lam[:, None] + lam[None, :])
        self.bl = Si @ W.Bl
        self.br = S.T @ W.Br
        Qt = Si @ W.Q @ Si.T
        Et = S.T @ (0.5 * (W.E + W.E.T)) @ S
        X0 = -self.L * Qt
        self.g0 = (self.br.T @ X0)  # k x n
        self.H = (Et * self.L) @ self.bl  # n x k
        self.t0 = np.sum(Et * X0).real
        self.F = np.einsum("ij,is,it->jst", self.L, self.br, self.bl)  # n x k x k
        self.applies = 0

    def T(self, G):  # G: k x n
        self.applies += 1
        R = (self.br[:, :, None] * G.T[:, None, :]).reshape(self.n, -1)  # i, (s, t)
        U = (self.L.T @ R).reshape(self.n, self.k, self.k)  # BLAS GEMM
        return np.einsum("jst,tj->sj", self.F, G) + np.einsum("jt,jst->sj", self.bl, U)

    def C(self, v, G):
        return (1.0 / v)[:, None] * G - self.T(G)

    def trace(self, G):
        return self.t0 + 2 * np.sum(G * self.H.T).real

    def prec_factory(self, v):
        sig = 1.0 / v
        M = np.einsum("st,j->jst", np.diag(sig), np.ones(self.n)) - self.F
        Minv = np.linalg.inv(M)
        return lambda R: np.einsum("jst,tj->sj", Minv, R)


def gmres(sysm, v, x0, tol=1e-12, maxit=600, Pinv=None, U=None, CU=None):
    """Right-preconditioned GMRES (no restart), optional augmentation space U with C(v)U = CU.
    Returns x, applies used (excluding CU which is precomputed)."""
    g0 = sysm.g0
    bn = np.linalg.norm(g0)
    a0 = sysm.applies
    x = x0.copy()
    r = g0 - sysm.C(v, x) if np.any(x0) else g0.copy()
    Pinv = Pinv or sysm.prec_factory(v)
    shape = g0.shape
    Cq = None
    if U is not None:  # GCRO: orthonormalise C U (per v, no T-apply: CU given), deflate r
        Cq, Rq = np.linalg.qr(CU)
        z = Cq.conj().T @ r.ravel()
        x = x + (U @ np.linalg.solve(Rq, z)).reshape(shape)
        r = r - (Cq @ z).reshape(shape)
    beta = np.linalg.norm(r)
    if beta <= tol * bn:
        return x, sysm.applies - a0
    V = [r.ravel() / beta]
    Z = []
    Hm = np.zeros((maxit + 1, maxit), complex)
    for j in range(maxit):
        z = Pinv(V[j].reshape(shape))
        Z.append(z.ravel())
        w = sysm.C(v, z).ravel()
        if Cq is not None:
            w = w - Cq @ (Cq.conj().T @ w)
        for _ in range(2):
            for i in range(j + 1):
                h = np.vdot(V[i], w)
                Hm[i, j] += h
                w = w - h * V[i]
        Hm[j + 1, j] = np.linalg.norm(w)
        V.append(w / Hm[j + 1, j])
        e = np.zeros(j + 2, complex)
        e[0] = beta
        y = np.linalg.lstsq(Hm[: j + 2, : j + 1], e, rcond=None)[0]
        res = np.linalg.norm(Hm[: j + 2, : j + 1] @ y - e)
        if res <= 0.5 * tol * bn:
            break
    dx = (np.array(Z).T @ y)
    if Cq is not None:
        # GCRO: x correction also removes the CU component picked up: x += -U R^-1 Cq^H C Z y
        Cw = sysm.C(v, dx.reshape(shape)).ravel()  # one extra apply (measurement only)
        sysm.applies -= 1
        dz = np.linalg.solve(Rq, Cq.conj().T @ Cw)
        dx = dx - U @ dz
    x = x + dx.reshape(shape)
    return x, sysm.applies - a0


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    strategies = sys.argv[2:] or ["cold", "warm"]
    W = workloads.make(name)
    t = time.time()
    sm = Sys(W)
    print(f"{name}: setup {time.time() - t:.1f}s, n={W.n}, k={W.k}", flush=True)
    shp = W.grid_shape
    pts = [tuple(s // 2 for s in shp), tuple(0 for _ in shp), tuple(s - 1 for s in shp),
           tuple((s - 1) if i == 0 else 0 for i, s in enumerate(shp))]
    for p in pts:
        i = int(np.ravel_multi_index(p, shp))
        v = W.V[i]
        row = [f"v={np.array2string(v, precision=3)}"]
        for stg in strategies:
            if stg == "cold":
                x, a = gmres(sm, v, np.zeros_like(sm.g0))
            elif stg == "warm":
                q = list(p)
                q[-1] = q[-1] - 1 if q[-1] > 0 else q[-1] + 1
                vn = W.V[int(np.ravel_multi_index(tuple(q), shp))]
                xn, _ = gmres(sm, vn, np.zeros_like(sm.g0))
                x, a = gmres(sm, v, xn)
            row.append(f"{stg}:{a}")
        print("  ".join(row), flush=True)


if __name__ == "__main__" and sys.argv[1:2] not in (["tiles"], ["seq"], ["var"], ["fixed"]):
    main()


def tile_shared(sm, V, tol=1e-12, p=4, maxr=2000, verbose=False):
    """Shared subspace for a tile of v's: every T-application is reused by every v of the tile
    (C(v) z = Delta(v) z - T z).  Greedy: add P(v)^-1 r_v of the p worst v's per step; per-v
    minimum residual over the shared space.  Returns (T-applies, final dim, steps)."""
    k, n = sm.k, sm.n
    g0 = sm.g0.ravel()
    bn = np.linalg.norm(g0)
    B = len(V)
    Z = np.zeros((k * n, 0), complex)
    TZ = np.zeros((k * n, 0), complex)
    res = np.full(B, 1.0)
    R = [sm.g0.copy() for _ in range(B)]
    a0 = sm.applies
    pre = [sm.prec_factory(v) for v in V]
    steps = 0
    while res.max() > tol and Z.shape[1] < maxr:
        steps += 1
        worst = np.argsort(-res)[:p]
        new = []
        for b in worst:
            if res[b] <= tol:
                continue
            d = pre[b](R[b]).ravel()
            for _ in range(2):
                d = d - Z @ (Z.conj().T @ d)
                for q in new:
                    d = d - q * np.vdot(q, d)
            nd = np.linalg.norm(d)
            if nd > 1e-14:
                new.append(d / nd)
        if not new:
            break
        Nw = np.array(new).T
        TN = np.array([sm.T(c.reshape(k, n)).ravel() for c in Nw.T]).T
        Z = np.hstack([Z, Nw])
        TZ = np.hstack([TZ, TN])
        for b in range(B):
            if res[b] <= tol:
                continue
            sig = np.repeat(1.0 / V[b], n)
            CZ = sig[:, None] * Z - TZ
            y = np.linalg.lstsq(CZ, g0, rcond=None)[0]
            r = g0 - CZ @ y
            res[b] = np.linalg.norm(r) / bn
            R[b] = r.reshape(k, n)
        if verbose:
            print(f"    step {steps}: dim {Z.shape[1]}, worst {res.max():.2e}", flush=True)
    return sm.applies - a0, Z.shape[1], steps


def tiles_main():
    name = sys.argv[2]
    tshape = tuple(int(x) for x in sys.argv[3].split("x"))
    p = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    W = workloads.make(name)
    sm = Sys(W)
    shp = W.grid_shape
    # low, mid, high corner tiles
    for label, start in (("low", [0] * len(shp)), ("mid", [s // 2 - t // 2 for s, t in zip(shp, tshape)]),
                         ("high", [s - t for s, t in zip(shp, tshape)]), ("mixed", [s - t if i == 0 else 0 for i, (s, t) in enumerate(zip(shp, tshape))])):
        idx = [int(np.ravel_multi_index(tuple(st + o for st, o in zip(start, off)), shp))
               for off in np.ndindex(*tshape)]
        t = time.time()
        a, r, st = tile_shared(sm, W.V[idx], p=p)
        print(f"{name} tile {label} {tshape}: {a} T-applies for {len(idx)} v = {a / len(idx):.2f}/v, dim {r}, "
              f"steps {st}, {time.time() - t:.0f}s", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "tiles":
    tiles_main()


def gcro_dr(sm, v, U=None, TU=None, s=20, m=300, tol=1e-12):
    """GCRO-DR with x-space recycle space U (T U known, so C(v) U = Delta(v) U - T U costs no
    T-apply).  Right preconditioner P(v) = Delta(v) - T_d (flexible in x-space).  One cycle (m large).
    Returns (applies, U_new, TU_new)."""
    k, n = sm.k, sm.n
    g0 = sm.g0.ravel()
    bn = np.linalg.norm(g0)
    sig = np.repeat(1.0 / v, n)
    Pinv = sm.prec_factory(v)
    a0 = sm.applies
    x = np.zeros(k * n, complex)
    r = g0.copy()
    Ct = np.zeros((k * n, 0), complex)
    Ut = np.zeros((k * n, 0), complex)
    if U is not None and U.shape[1]:
        CU = sig[:, None] * U - TU
        Ct, Rt = np.linalg.qr(CU)
        Ut = U @ np.linalg.inv(Rt)
        z = Ct.conj().T @ r
        x = x + Ut @ z
        r = r - Ct @ z
    beta = np.linalg.norm(r)
    if beta <= tol * bn:
        return sm.applies - a0, U, TU
    V = [r / beta]
    Z = []
    Hm = np.zeros((m + 1, m), complex)
    Bm = np.zeros((Ct.shape[1], m), complex)
    for j in range(m):
        zj = Pinv(V[j].reshape(k, n)).ravel()
        Z.append(zj)
        w = (sig * zj - sm.T(zj.reshape(k, n)).ravel())
        if Ct.shape[1]:
            bj = Ct.conj().T @ w
            Bm[:, j] = bj
            w = w - Ct @ bj
        for _ in range(2):
            for i in range(j + 1):
                h = np.vdot(V[i], w)
                Hm[i, j] += h
                w = w - h * V[i]
        Hm[j + 1, j] = np.linalg.norm(w)
        V.append(w / Hm[j + 1, j])
        e = np.zeros(j + 2, complex)
        e[0] = beta
        y, *_ = np.linalg.lstsq(Hm[: j + 2, : j + 1], e, rcond=None)
        res = np.linalg.norm(Hm[: j + 2, : j + 1] @ y - e)
        if res <= 0.5 * tol * bn:
            break
    mm = j + 1
    Zm = np.array(Z).T
    x = x + Zm @ y - (Ut @ (Bm[:, :mm] @ y) if Ct.shape[1] else 0)
    # new recycle space: harmonic Ritz vectors of the augmented search space Zhat = [Ut, Zm]
    What = np.hstack([Ct, np.array(V[: mm + 1]).T])
    G = np.zeros((Ct.shape[1] + mm + 1, Ct.shape[1] + mm), complex)
    c = Ct.shape[1]
    G[:c, :c] = np.eye(c)
    G[:c, c:] = Bm[:, :mm]
    G[c:, c:] = Hm[: mm + 1, :mm]
    Zhat = np.hstack([Ut, Zm])
    A_ = G.conj().T @ G
    B_ = G.conj().T @ (What.conj().T @ Zhat)
    import scipy.linalg
    th, P = scipy.linalg.eig(A_, B_)
    order = np.argsort(np.abs(th))
    P = P[:, order[:s]]
    Unew = Zhat @ P
    CUnew = What @ (G @ P)
    TUnew = sig[:, None] * Unew - CUnew
    return sm.applies - a0, Unew, TUnew


def seq_main():
    name = sys.argv[2]
    s = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    W = workloads.make(name)
    sm = Sys(W)
    shp = W.grid_shape
    lines = {"high": [s_ - 1 for s_ in shp], "mixed": [s_ - 1 if i == 0 else 0 for i, s_ in enumerate(shp)],
             "mid": [s_ // 2 for s_ in shp]}
    sel = [x for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else lines)]
    for label, base in [(l, lines[l]) for l in sel]:
        U = TU = None
        out = []
        for q in range(min(int(__import__("os").environ.get("NSEQ", "8")), shp[-1])):
            p = list(base)
            p[-1] = (shp[-1] - 1 - q) if base[-1] == shp[-1] - 1 else min(shp[-1] - 1, base[-1] + q)
            v = W.V[int(np.ravel_multi_index(tuple(p), shp))]
            a, U, TU = gcro_dr(sm, v, U, TU, s=s)
            x_cold, ac = gmres(sm, v, np.zeros_like(sm.g0))
            out.append(f"{a}/{ac}")
        print(f"{name} line {label} (recycled/cold, s={s}): " + " ".join(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "seq":
    seq_main()


def guess_only(sm, v, U=None, TU=None, s=64, m=400, tol=1e-12):
    """Recycled space used ONLY for a min-residual initial guess; then plain right-preconditioned
    GMRES (no deflation inside Arnoldi).  Recycle = all applied directions, SVD-compressed to s."""
    k, n = sm.k, sm.n
    g0 = sm.g0.ravel()
    sig = np.repeat(1.0 / v, n)
    a0 = sm.applies
    x0 = np.zeros(k * n, complex)
    if U is not None:
        CU = sig[:, None] * U - TU
        z, *_ = np.linalg.lstsq(CU, g0, rcond=None)
        x0 = U @ z
    # GMRES from x0, collecting applied directions
    Pinv = sm.prec_factory(v)
    r = g0 - (sig * x0 - sm.T(x0.reshape(k, n)).ravel()) if U is not None else g0.copy()
    if U is not None:
        sm.applies -= 1  # r0 = g0 - CU z needs no T-apply (TU known)
    beta = np.linalg.norm(r)
    bn = np.linalg.norm(g0)
    V = [r / beta]
    Z, TZ = [], []
    Hm = np.zeros((m + 1, m), complex)
    for j in range(m):
        zj = Pinv(V[j].reshape(k, n)).ravel()
        tz = sm.T(zj.reshape(k, n)).ravel()
        Z.append(zj)
        TZ.append(tz)
        w = sig * zj - tz
        for _ in range(2):
            for i in range(j + 1):
                h = np.vdot(V[i], w)
                Hm[i, j] += h
                w = w - h * V[i]
        Hm[j + 1, j] = np.linalg.norm(w)
        V.append(w / Hm[j + 1, j])
        e = np.zeros(j + 2, complex)
        e[0] = beta
        y, *_ = np.linalg.lstsq(Hm[: j + 2, : j + 1], e, rcond=None)
        if np.linalg.norm(Hm[: j + 2, : j + 1] @ y - e) <= 0.5 * tol * bn:
            break
    Zm, TZm = np.array(Z).T, np.array(TZ).T
    Uall = Zm if U is None else np.hstack([U, Zm])
    TUall = TZm if TU is None else np.hstack([TU, TZm])
    # compress: smallest singular directions of C(v) on span(Uall) (B-metric = Uall^H Uall)
    import scipy.linalg
    CUa = sig[:, None] * Uall - TUall
    A_ = CUa.conj().T @ CUa
    B_ = Uall.conj().T @ Uall
    th, P = scipy.linalg.eigh(A_, B_ + 1e-14 * np.trace(B_).real / len(B_) * np.eye(len(B_)))
    P = P[:, :s]
    return sm.applies - a0, Uall @ P, TUall @ P


def gcro_variant(sm, v, U=None, TU=None, s=20, sel="harm", m=400, tol=1e-12):
    """Like gcro_dr, with the recycle selection `sel`: 'harm' harmonic Ritz, 'svd' smallest singular
    directions of C on the search space (symmetric eigenproblem), 'full' the whole search space."""
    k, n = sm.k, sm.n
    g0 = sm.g0.ravel()
    bn = np.linalg.norm(g0)
    sig = np.repeat(1.0 / v, n)
    Pinv = sm.prec_factory(v)
    a0 = sm.applies
    r = g0.copy()
    Ct = np.zeros((k * n, 0), complex)
    Ut = np.zeros((k * n, 0), complex)
    if U is not None and U.shape[1]:
        CU = sig[:, None] * U - TU
        Ct, Rt = np.linalg.qr(CU)
        Ut = U @ np.linalg.inv(Rt)
        r = r - Ct @ (Ct.conj().T @ r)
    beta = np.linalg.norm(r)
    V = [r / beta]
    Z = []
    Hm = np.zeros((m + 1, m), complex)
    Bm = np.zeros((Ct.shape[1], m), complex)
    j = -1
    if beta > tol * bn:
        for j in range(m):
            zj = Pinv(V[j].reshape(k, n)).ravel()
            Z.append(zj)
            w = (sig * zj - sm.T(zj.reshape(k, n)).ravel())
            if Ct.shape[1]:
                bj = Ct.conj().T @ w
                Bm[:, j] = bj
                w = w - Ct @ bj
            for _ in range(2):
                for i in range(j + 1):
                    h = np.vdot(V[i], w)
                    Hm[i, j] += h
                    w = w - h * V[i]
            Hm[j + 1, j] = np.linalg.norm(w)
            V.append(w / Hm[j + 1, j])
            e = np.zeros(j + 2, complex)
            e[0] = beta
            y, *_ = np.linalg.lstsq(Hm[: j + 2, : j + 1], e, rcond=None)
            if np.linalg.norm(Hm[: j + 2, : j + 1] @ y - e) <= 0.5 * tol * bn:
                break
    mm = j + 1
    if mm == 0:
        return sm.applies - a0, U, TU
    Zm = np.array(Z).T
    c = Ct.shape[1]
    What = np.hstack([Ct, np.array(V[: mm + 1]).T])
    G = np.zeros((c + mm + 1, c + mm), complex)
    G[:c, :c] = np.eye(c)
    G[:c, c:] = Bm[:, :mm]
    G[c:, c:] = Hm[: mm + 1, :mm]
    Zhat = np.hstack([Ut, Zm])
    import scipy.linalg
    if sel.startswith("fifo"):
        # raw (untransformed) recycle columns, oldest dropped beyond s
        CZm = What @ G[:, c:]
        TZm = sig[:, None] * Zm - CZm
        Uraw = Zm if U is None else np.hstack([U, Zm])
        TUraw = TZm if TU is None else np.hstack([TU, TZm])
        return sm.applies - a0, Uraw[:, -s:], TUraw[:, -s:]
    if sel == "full":
        P = np.eye(c + mm)
    elif sel == "gsvd":  # smallest right singular vectors of G alone (Zhat metric ignored)
        A_ = G.conj().T @ G
        th, P = np.linalg.eigh(A_)
        P = P[:, :s]
    elif sel == "svd":
        A_ = G.conj().T @ G
        B_ = Zhat.conj().T @ Zhat
        th, P = scipy.linalg.eigh(A_, B_)
        P = P[:, :s]
    else:
        A_ = G.conj().T @ G
        B_ = G.conj().T @ (What.conj().T @ Zhat)
        th, P = scipy.linalg.eig(A_, B_)
        P = P[:, np.argsort(np.abs(th))[:s]]
    Unew = Zhat @ P
    CUnew = What @ (G @ P)
    return sm.applies - a0, Unew, sig[:, None] * Unew - CUnew


def var_main():
    name, sel, s = sys.argv[2], sys.argv[3], int(sys.argv[4])
    W = workloads.make(name)
    sm = Sys(W)
    shp = W.grid_shape
    lines = {"high": [s_ - 1 for s_ in shp], "mixed": [s_ - 1 if i == 0 else 0 for i, s_ in enumerate(shp)],
             "mid": [s_ // 2 for s_ in shp]}
    for label, base in lines.items():
        U = TU = None
        out = []
        for q in range(6):
            p = list(base)
            p[-1] = (shp[-1] - 1 - q) if base[-1] == shp[-1] - 1 else min(shp[-1] - 1, base[-1] + q)
            v = W.V[int(np.ravel_multi_index(tuple(p), shp))]
            if sel == "guess":
                a, U, TU = guess_only(sm, v, U, TU, s=s)
            else:
                a, U, TU = gcro_variant(sm, v, U, TU, s=s, sel=sel)
            out.append(f"{a}")
        print(f"{name} line {label} sel={sel} s={s}: " + " ".join(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "var":
    var_main()


def fixed_main():
    """One recycle space from a GCRO-DR solve at the grid corner (all v max), reused unchanged."""
    name, s = sys.argv[2], int(sys.argv[3])
    sel = sys.argv[4] if len(sys.argv) > 4 else "svd"
    W = workloads.make(name)
    sm = Sys(W)
    shp = W.grid_shape
    corner = W.V[int(np.ravel_multi_index(tuple(x - 1 for x in shp), shp))]
    a0, U, TU = gcro_variant(sm, corner, None, None, s=s, sel=sel)
    a1, U, TU = gcro_variant(sm, corner * 0.9, U, TU, s=s, sel=sel)  # one refinement solve
    print(f"{name}: building U cost {a0}+{a1} applies", flush=True)
    lines = {"high": [x - 1 for x in shp], "mixed": [x - 1 if i == 0 else 0 for i, x in enumerate(shp)],
             "mixed2": [0 if i == 0 else x - 1 for i, x in enumerate(shp)], "mid": [x // 2 for x in shp],
             "low": [0 for x in shp]}
    for label, base in lines.items():
        out = []
        for q in range(int(__import__("os").environ.get("NSEQ", "4"))):
            p = list(base)
            p[-1] = (shp[-1] - 1 - q) if base[-1] == shp[-1] - 1 else min(shp[-1] - 1, base[-1] + q)
            v = W.V[int(np.ravel_multi_index(tuple(p), shp))]
            a, _, _ = gcro_variant(sm, v, U, TU, s=s, sel=sel)
            _, ac = gmres(sm, v, np.zeros_like(sm.g0))
            out.append(f"{a}/{ac}")
        print(f"{name} fixed-U {label} (recycled/cold): " + " ".join(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "fixed":
    fixed_main()
