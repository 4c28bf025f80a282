"""Exploration: per-v T-applies on a config (diagnostics of trace_batch) and an LPT simulation of the
lock-step slot schedule (makespan vs the ideal total / b).  python tools/explore/c5_applies.py c5 [b]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import workloads  # noqa: E402
from paper_2312_08201_b200 import Problem  # noqa: E402

name = sys.argv[1]
W = workloads.make(name)
P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E, device=0)
tau, st, ap, rs = P.trace_batch(W.V, return_diagnostics=True)
P.reset_stats()
P.trace_batch(torch.tensor(W.V, device="cuda"))
s = P.stats
print("batch", P.info["batch"], "iterations", s["iterations"], "k1_vectors", s["k1_vectors"], "launches", s["k1_launches"])
np.save(f"gpurun_out/applies_{name}.npy", ap)
print("applies/v mean %.2f max %d" % (ap.mean(), ap.max()))
q = np.percentile(ap, [10, 25, 50, 75, 90, 99])
print("percentiles 10/25/50/75/90/99:", q)
cost = P.cost_proxy(W.V)
order = np.argsort(-cost, kind="stable")
for b in (296, 444, 592, 888, 1184):
    G = 2
    per = b // G
    # LPT per group over a shared queue (dynamic): each free slot takes the next v; +2 iterations per v
    import heapq
    slots = [(0, i) for i in range(b)]
    heapq.heapify(slots)
    for idx in order:
        t, i = heapq.heappop(slots)
        heapq.heappush(slots, (t + ap[idx] + 2, i))
    mk = max(t for t, _ in slots)
    print(f"b={b}: ideal {ap.sum() / b:.0f} its, LPT makespan {mk} its, fill {ap.sum() / (b * mk):.2f}")
