"""Small workload for compute-sanitizer: engine (1 and 2 slot groups), K1 apply, v=0, negative v."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import workloads  # noqa: E402
from paper_2312_08201_b200 import Problem  # noqa: E402

rng = np.random.default_rng(1)
A0, Bl, Br, Q, E = workloads.random_stable(37, 3, rng, shift=2.0)
V = rng.uniform(0.05, 2.0, (70, 3))
V[3] = [0.0, 0.4, 1.0]
V[5] = [-0.2, 0.3, 0.1]
for batch in (8, 64):
    P = Problem(A0, Bl, Br, Q, E, batch=batch, max_dim=40)
    t = P.trace_batch(V)
    X = torch.randn(5, 3, P.info["npad"], dtype=torch.float64, device="cuda")
    X[:, :, 37:] = 0
    Y = P.apply_C(X, torch.rand(5, 3, dtype=torch.float64, device="cuda"))
    P.close()
W = workloads.make("c1")
P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E)
t = P.trace_batch(W.V[:40])
print("ok", float(t[0]))
