"""Write tests/golden/oracle_<cfg>.json: CPU-oracle traces on seeded samples of each config.

Calls only workloads/ (inputs) and oracle/ (the Bartels-Stewart oracle). Each sample holds the
2^k grid corners, the grid centre and a seeded uniform draw (Workload.sample_indices).
Usage: python tools/make_golden.py [c1 c2 ...]   (parallel over processes, 1 BLAS thread each)
"""
import json
import os
import pathlib
import sys
import time

for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[var] = "1"
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402

SAMPLES = {"c1": 256, "c2": 256, "c3": 256, "c4": 64, "c5": 32}
_W = {}


def _work(args):
    name, idx = args
    if name not in _W:
        _W[name] = workloads.make(name)
    W = _W[name]
    t = time.time()
    tau, d = oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[idx], diagnostics=True)
    return idx, tau, d["residual"], d["backward_error"], time.time() - t


def main(names):
    procs = int(os.environ.get("GOLDEN_PROCS", os.cpu_count() or 1))
    for name in names:
        W = workloads.make(name)
        idx = [int(i) for i in W.sample_indices(SAMPLES[name], seed=0)] if SAMPLES[name] < W.nv \
            else list(range(W.nv))
        t0 = time.time()
        with mp.Pool(procs) as pool:
            res = pool.map(_work, [(name, i) for i in idx], chunksize=1)
        res.sort()
        doc = {
            "config": name, "seed": W.meta["seed"], "n": W.n, "k": W.k, "nv": W.nv,
            "generator": "workloads.make(%r)" % name, "oracle": "oracle.trace_EX (blocked Bartels-Stewart)",
            "indices": [r[0] for r in res], "V": [W.V[r[0]].tolist() for r in res],
            "traces": [r[1] for r in res], "residual": [r[2] for r in res],
            "backward_error": [r[3] for r in res], "seconds_per_v": [r[4] for r in res],
        }
        (ROOT / "tests" / "golden" / f"oracle_{name}.json").write_text(json.dumps(doc, indent=0))
        print(name, len(idx), "samples in %.1fs" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SAMPLES))
