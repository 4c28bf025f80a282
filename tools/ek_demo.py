"""NEXT row f1 demonstration (GPU): the extended-Krylov projection (§2.2, Alg. 1) with per-v
certification on the configurations where the space compresses -- c3 (multi-agent, the paper's
Ex. 2/3 setting) and c5 (chain n = 4000, the paper's Ex. 1b scale) --
against the oracle goldens and beside the dense engine on the same v.

The seed solution X0 that P = [X0 Br, Bl] needs: c5 from the closed form of the modal chain (reading
R1: per mode [[1/c + c/(2w^2), -1/(2w)], [-1/(2w), 1/c]], c = 2 alpha w, Q = I), c3 from SciPy.

python tools/ek_demo.py [c3 c5] [--eps 1e-8] > gpurun_out/ek_demo.json
"""
import argparse
import json
import pathlib
import sys
import time

import numpy as np
import scipy.linalg

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import workloads  # noqa: E402
from paper_2312_08201_b200 import EKProblem, Problem  # noqa: E402


def chain_X0(A0):
    """Closed-form seed Gramian of the modal chain A0 = [[0, W], [-W, -2 a W]] with Q = I."""
    n = A0.shape[0]
    m = n // 2
    X0 = np.zeros((n, n))
    for i in range(m):
        w = A0[i, m + i]
        c = -A0[m + i, m + i]
        X0[i, i] = 1.0 / c + c / (2 * w * w)
        X0[i, m + i] = X0[m + i, i] = -1.0 / (2 * w)
        X0[m + i, m + i] = 1.0 / c
    return X0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["c3", "c5"])
    ap.add_argument("--eps", type=float, default=1e-8)
    args = ap.parse_args()
    # the closed form, checked on a small chain against SciPy
    Ws = workloads.chain(20, 300.0, 0.01, [3, 11])[0]
    Xs = scipy.linalg.solve_continuous_lyapunov(Ws, -np.eye(Ws.shape[0]))
    assert np.abs(chain_X0(Ws) - Xs).max() <= 1e-9 * np.abs(Xs).max()
    out = []
    for name in args.names:
        W = workloads.make(name)
        g = json.loads((ROOT / "tests" / "golden" / f"oracle_{name}.json").read_text())
        idx = np.array(g["indices"])
        ref = np.array(g["traces"])
        t = time.perf_counter()
        X0 = chain_X0(W.A0) if name in ("c1", "c2", "c5") else scipy.linalg.solve_continuous_lyapunov(W.A0, -W.Q)
        t_x0 = time.perf_counter() - t
        t0 = float(np.sum(0.5 * (W.E + W.E.T) * X0))
        t = time.perf_counter()
        ek = EKProblem(W.A0, W.Bl, W.Br, X0 @ W.Br, W.E, t0, max_dim=W.n)
        t_setup = time.perf_counter() - t
        t = time.perf_counter()
        tau, bwd, dim = ek.trace_batch(W.V[idx], eps=args.eps, per_v=True, allow_partial=True)
        t_ek = time.perf_counter() - t
        ek.close()
        err = np.abs(tau - ref) / np.abs(ref)
        t = time.perf_counter()
        P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E)
        t_dense_setup = time.perf_counter() - t
        t = time.perf_counter()
        taud = P.trace_batch(W.V[idx])
        t_dense = time.perf_counter() - t
        P.close()
        rec = {"config": name, "n": W.n, "k": W.k, "nv": int(len(idx)), "eps": args.eps,
               "x0_s": t_x0, "ek_setup_s": t_setup, "ek_trace_s": t_ek,
               "dim_min": int(dim.min()), "dim_max": int(dim.max()), "dim_mean": float(dim.mean()),
               "bwd_max": float(bwd.max()), "certified": int(np.sum(bwd <= args.eps)),
               "rel_err_max": float(err.max()), "rel_err_median": float(np.median(err)),
               "dense_setup_s": t_dense_setup, "dense_trace_s": t_dense,
               "dense_rel_err_max": float(np.max(np.abs(taud - ref) / np.abs(ref)))}
        print(json.dumps(rec), flush=True)
        out.append(rec)


if __name__ == "__main__":
    main()
