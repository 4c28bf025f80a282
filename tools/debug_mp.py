"""Diagnostics: c5 golden samples with mixed precision (env LYAP_MP_FUSE selects the fused epilogues)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2312_08201_b200 import Problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
g = json.load(open(f"tests/golden/oracle_{name}.json"))
W = workloads.make(name)
idx = np.array(g["indices"])
P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E, device=0, mixed=1)
tau, st, ap, rs = P.trace_batch(torch.tensor(W.V[idx], device="cuda:0"), return_diagnostics=True)
tau = tau.cpu().numpy()
err = np.abs(tau - np.array(g["traces"])) / np.abs(np.array(g["traces"]))
print(name, "fuse", os.environ.get("LYAP_MP_FUSE", "3"), "max rel err", err.max(), "status", np.unique(st.cpu().numpy() if hasattr(st, "cpu") else st),
      "applies", float(np.mean(ap.cpu().numpy() if hasattr(ap, "cpu") else ap)), "stats", P.stats["k1_exact_vectors"], P.stats["k1_vectors"])
