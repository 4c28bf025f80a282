"""Profiling window for ncu (--profile-from-start off): set up a BASELINE configuration, solve the
grid once untimed (warm-up: coarse space, graphs, Lf32), then run one trace_batch of the whole grid
between cudaProfilerStart / cudaProfilerStop.  Not a bench: ncu times are serialised, cold-cache.

python tools/profile_step.py c5 [--mixed M] [--nv NV]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2312_08201_b200 import Problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--mixed", type=int, default=-1)
ap.add_argument("--nv", type=int, default=0)
args = ap.parse_args()
W = workloads.make(args.config)
V = torch.tensor(W.V if args.nv <= 0 else W.V[:: max(1, W.nv // args.nv)][: args.nv], device="cuda:0")
P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E, device=0, mixed=args.mixed)
P.trace_batch(V)
torch.cuda.synchronize()
torch.cuda.profiler.start()
P.trace_batch(V)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("stats", P.stats)
P.close()
