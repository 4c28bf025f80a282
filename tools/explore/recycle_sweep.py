"""Exploration: applies/v and v/s of the per-v engine with recycle spaces from different seed sets.
python tools/explore/recycle_sweep.py c5 [reps]"""
import itertools
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import workloads  # noqa: E402
from paper_2312_08201_b200 import Problem  # noqa: E402


def seeds_grid(V, per_axis):
    lo, hi = V.min(0), V.max(0)
    axes = [np.geomspace(l, h, per_axis) for l, h in zip(lo, hi)]
    return np.array(list(itertools.product(*axes)))


def run(P, Vd, label):
    P.trace_batch(Vd)
    torch.cuda.synchronize()
    P.reset_stats()
    t = time.perf_counter()
    tau = P.trace_batch(Vd)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    st = P.stats
    print(f"{label}: {Vd.shape[0] / el:.1f} v/s  applies/v {st['k1_vectors'] / Vd.shape[0]:.2f}  "
          f"build {st['recycle_build_ms']:.0f} ms", flush=True)
    return tau


def main():
    name = sys.argv[1]
    W = workloads.make(name)
    Vd = torch.tensor(W.V, device="cuda")
    cfgs = [("off", 0, None), ("corners s32", 32, 2), ("3^k s32", 32, 3), ("3^k s48", 48, 3), ("corners s64", 64, 2)]
    ref = None
    for label, s, per in cfgs:
        P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E, recycle=0, device=0)
        if s:
            t = time.perf_counter()
            P.build_recycle(seeds=seeds_grid(W.V, per), s=s)
            print(f"  build {label}: {1e3 * (time.perf_counter() - t):.0f} ms", flush=True)
        tau = run(P, Vd, label).cpu().numpy()
        if ref is None:
            ref = tau
        else:
            print(f"  max rel diff vs off: {np.max(np.abs(tau - ref) / np.abs(ref)):.2e}")
        P.close()


if __name__ == "__main__":
    main()
