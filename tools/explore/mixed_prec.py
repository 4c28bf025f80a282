"""Exploration (not product code): mixed-precision GMRES for C(v) g = g0.

Inner Krylov steps apply T with the dense Cauchy GEMM in reduced precision (fp32, or tf32 inputs with
fp32 accumulation, or 3xtf32 split); every restart recomputes the TRUE residual with the exact FP64
T (iterative refinement: each cycle solves C(v) d = r to a relative reduction eta).  Counts inner
(low-precision) and exact applies to a true residual <= tol.

python tools/explore/mixed_prec.py c2 fp32,tf32 1e-4,1e-6 high,p80,mid,mixed [m]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/", 1)[0])
import workloads  # noqa: E402
from tile_galerkin import Sys  # noqa: E402


def tf32(x):
    """round fp32 tensor (real) to tf32 (10-bit mantissa, round to nearest even-ish)"""
    i = x.view(torch.int32)
    i = (i + 0x1000) & ~0x1FFF
    return i.view(torch.float32)


def ctf32(z):
    return torch.complex(tf32(z.real.contiguous()), tf32(z.imag.contiguous()))


class LowT:
    def __init__(self, sm, mode):
        self.sm, self.mode = sm, mode
        LT = sm.LT
        if mode == "fp32":
            self.A = LT.to(torch.complex64)
        elif mode == "tf32":
            self.A = ctf32(LT.to(torch.complex64))
        elif mode == "3xtf32":
            a32 = LT.to(torch.complex64)
            self.Ah = ctf32(a32)
            self.Al = ctf32(a32 - self.Ah)
        self.applies = 0

    def __call__(self, G):
        sm = self.sm
        p = G.shape[0]
        self.applies += p
        R = (sm.br[:, None, :, None] * G.permute(2, 0, 1)[:, :, None, :]).reshape(sm.n, -1)
        if self.mode == "fp32":
            U = (self.A @ R.to(torch.complex64)).to(torch.complex128)
        elif self.mode == "tf32":
            U = (self.A @ ctf32(R.to(torch.complex64))).to(torch.complex128)
        else:
            r32 = R.to(torch.complex64)
            rh = ctf32(r32)
            rl = ctf32(r32 - rh)
            U = (self.Ah @ rh + (self.Ah @ rl + self.Al @ rh)).to(torch.complex128)
        U = U.reshape(sm.n, p, sm.k, sm.k)
        return torch.einsum("jst,btj->bsj", sm.F, G) + torch.einsum("jt,jbst->bsj", sm.bl, U)


def solve(sm, v, Tlow, eta, tol=1e-12, m=400, max_cycles=60):
    dev = sm.dev
    k, n = sm.k, sm.n
    Vt = torch.tensor(v[None], device=dev)
    Pm = sm.pminv(Vt)
    ap = lambda R: sm.papply(Pm, R)  # noqa: E731
    sig = (1.0 / Vt).to(torch.complex128).repeat_interleave(n, dim=1)[0]
    g0 = sm.g0.reshape(-1)
    bn = torch.linalg.norm(g0).item()
    x = torch.zeros_like(g0)
    a0 = sm.applies
    inner = 0
    cyc = 0
    hist = []
    Cop_low = (lambda z: sig * z.reshape(-1) - Tlow(z).reshape(-1)) if Tlow is not None else \
        (lambda z: sig * z.reshape(-1) - sm.T(z).reshape(-1))
    while cyc < max_cycles:
        r = g0 - (sig * x - sm.T(x.reshape(1, k, n)).reshape(-1)) if cyc else g0.clone()
        rn = torch.linalg.norm(r).item()
        hist.append(rn / bn)
        if rn <= tol * bn:
            break
        cyc += 1
        target = max(eta * rn, 0.5 * tol * bn)
        beta = rn
        Qb = [r / beta]
        Zs = []
        H = torch.zeros(m + 1, m, dtype=torch.complex128, device=dev)
        for j in range(m):
            z = ap(Qb[j].reshape(1, k, n))
            Zs.append(z.reshape(-1))
            w = Cop_low(z)
            inner += 1
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
            if torch.linalg.norm(H[: j + 2, : j + 1] @ y - e).item() <= target:
                break
        x = x + torch.stack(Zs, 1) @ y
    exact = sm.applies - a0
    return inner, exact, cyc, hist


def main():
    name = sys.argv[1]
    modes = sys.argv[2].split(",")
    etas = [float(e) for e in sys.argv[3].split(",")]
    which = sys.argv[4].split(",")
    m = int(sys.argv[5]) if len(sys.argv) > 5 else 400
    W = workloads.make(name)
    sm = Sys(W, "cpu")
    shp = W.grid_shape
    pts = {"low": [0] * len(shp), "high": [s - 1 for s in shp], "mid": [s // 2 for s in shp],
           "mixed": [s - 1 if i == 0 else 0 for i, s in enumerate(shp)], "p80": [int(0.8 * s) for s in shp]}
    for label in which:
        v = W.V[int(np.ravel_multi_index(tuple(pts[label]), shp))]
        t = time.time()
        inner, exact, cyc, hist = solve(sm, v, None, 1e-30, m=m)
        print(f"{name} {label} v={np.round(v, 3)} fp64 restart {m}: applies {inner} + verify {exact} "
              f"cycles {cyc} ({time.time() - t:.1f}s)", flush=True)
        for mode in modes:
            Tl = LowT(sm, mode)
            for eta in etas:
                t = time.time()
                inner, exact, cyc, hist = solve(sm, v, Tl, eta, m=m)
                print(f"   {mode} eta {eta:g}: inner {inner} exact {exact} cycles {cyc} final {hist[-1]:.1e} "
                      f"hist {' '.join(f'{h:.0e}' for h in hist[:8])} ({time.time() - t:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
