#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q -k "extended_krylov" > gpurun_out/z3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z_pytest.log
timeout 600 python - > gpurun_out/z3_ek.log 2>&1 <<'PY'
import sys, time, json, numpy as np, scipy.linalg
sys.path.insert(0, ".")
import workloads
from paper_2312_08201_b200 import EKProblem
for name in ("c1", "c2", "c4"):
    W = workloads.make(name)
    X0 = scipy.linalg.solve_continuous_lyapunov(W.A0, -W.Q)
    t0 = float(np.sum(W.E * X0))
    g = json.load(open(f"tests/golden/oracle_{name}.json"))
    idx = np.array(g["indices"]); ref = np.array(g["traces"])
    for eps in (1e-6, 1e-8, 1e-10):
        ek = EKProblem(W.A0, W.Bl, W.Br, X0 @ W.Br, W.E, t0, max_dim=800)
        t = time.time(); tau, dim, bwd = ek.trace_batch(W.V[idx], eps=eps); el = time.time() - t
        print(name, "eps", eps, "dim", dim, "bwd", bwd, "max rel err", float(np.max(np.abs(tau-ref)/np.abs(ref))), "s", round(el, 2), flush=True)
        ek.close()
PY
echo "rc=$?" >> gpurun_out/z3_ek.log
