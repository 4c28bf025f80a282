#!/usr/bin/env python
"""Benchmark: parameter vectors per second of trace(E X(v)) on B200 (BASELINE.json metric).

python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl reference]

A step = one lyap_trace_batch over the configuration's whole parameter grid (this rank's shard),
followed by the all-gather of traces and the argmin.  Inputs are synthetic and
seeded (workloads.make), resident in HBM before the timed region.  Multi-GPU: one process per GPU
(torchrun), the grid is split into chunks of consecutive grid points dealt round-robin to ranks
(strong scaling: the grid is fixed), NCCL all-gather of traces, max-over-ranks device time.

Only the `cpu_baseline` leg and `--impl reference` execute oracle/ (the CPU oracle); the timed
product path is liblyapgpu.so only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "parameter vectors/sec (trace(EX(v)))"
UNIT = "v/s"
FP64_PEAK_TFLOPS = 37.0   # measured: DMMA m8n8k4 burst, profiles/r01_fp64_peaks.md (MEASURED_PEAKS.json has no FP64)
TF32_PER_BF16 = 1.1 / 2.25  # B200_PROFILING.md nominal dense tf32 / bf16 tensor peaks


def bf16_peak():
    """FP16/BF16 dense tensor peak from MEASURED_PEAKS.json (fp16 runs at the bf16 rate).  The tcgen05 kernel is
    timed inside a long step (hundreds of back-to-back launches per second-long step, the board at its power
    cap), so the roofline denominator is the SUSTAINED figure; the burst one is reported beside it.
    Returns (peak, source, burst)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        burst = float(mp["bf16_tflops"])
        if "bf16_tflops_sustained" in mp:
            sus = float(mp["bf16_tflops_sustained"])
            return sus, (f"MEASURED_PEAKS.json bf16_tflops_sustained {sus:.1f} (kernel timed inside a long step; "
                         f"burst {burst:.1f}; dense fp16 = bf16 rate)"), burst
        return burst, f"MEASURED_PEAKS.json bf16_tflops {burst:.1f} (burst; dense fp16 = bf16 rate)", burst
    except (OSError, KeyError, ValueError):
        return 2250.0, "B200_PROFILING.md nominal dense bf16/fp16 2.25 PFLOP/s (MEASURED_PEAKS.json absent)", 2250.0


def tf32_peak():
    """TF32 dense tensor peak: MEASURED_PEAKS.json bf16 burst x the guide's nominal tf32/bf16 ratio."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        return bf16 * TF32_PER_BF16, f"MEASURED_PEAKS.json bf16_tflops {bf16:.1f} (burst) x {TF32_PER_BF16:.3f} " \
                                     "(B200_PROFILING.md nominal dense tf32 1.1 / bf16 2.25 PFLOP/s)"
    except (OSError, KeyError, ValueError):
        return 2250.0 * TF32_PER_BF16, "B200_PROFILING.md nominal dense tf32 1.1 PFLOP/s (MEASURED_PEAKS.json absent)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("BENCH_CONFIG", "c5"),
                    help="BASELINE configuration; default c5 = configs[4], the 1/2/4/8-GPU configuration the "
                         "metric is quoted on")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--scaling", default=os.environ.get("BENCH_SCALING", "strong"), choices=["weak", "strong"],
                    help="strong (default): the configuration's one grid is sharded over the ranks, cost-balanced "
                         "(BASELINE c5: 'sharded over 1/2/4/8 GPUs'); weak: every rank solves a full-size grid of "
                         "its own (axis 0 refined world-fold and interleaved; N=1 is the configuration itself)")
    ap.add_argument("--emulate-rank", default="",
                    help="R/N: on this single process, solve only rank R's shard of an N-way strong split "
                         "(per-rank time of an N-GPU run, measured on one GPU)")
    ap.add_argument("--max-dim", type=int, default=0)
    ap.add_argument("--no-profile", action="store_true", help="no per-launch K1 events (diagnostics)")
    ap.add_argument("--coarse", type=int, default=int(os.environ.get("BENCH_COARSE", "-1")),
                    help="two-level preconditioner coarse-space size (-1 auto, 0 off)")
    ap.add_argument("--mixed", type=int, default=int(os.environ.get("BENCH_MIXED", "-1")),
                    help="mixed-precision iterative refinement (-1 auto: n > 1536, 0 off, 1 on; DESIGN.md §2.8)")
    ap.add_argument("--mixed-eta", type=float, default=float(os.environ.get("BENCH_MIXED_ETA", "1e-4")),
                    help="residual reduction per mixed-precision refinement cycle")
    ap.add_argument("--recycle", type=int, default=int(os.environ.get("BENCH_RECYCLE", "0")),
                    help="recycle-space size s (0: off); spaces built from the 2^k grid corners before timing")
    return ap.parse_args()


# ------------------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling during the timed region (the B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.rows, self.proc = [], None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for nm, val in zip(names, r[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------ CPU oracle timing
_WK = {}


_THREAD_VARS = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "BLIS_NUM_THREADS")


def _oracle_worker_init(name):
    # one BLAS thread per worker process: the env is inherited from the parent (set before the
    # pool starts) and threadpoolctl re-limits every BLAS already loaded (numpy's and scipy's)
    import scipy.linalg  # noqa: F401  (load scipy's OpenBLAS before limiting)
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    import oracle  # noqa: F401
    import workloads
    _WK["W"] = workloads.make(name)


def _oracle_one(idx):
    import oracle
    W = _WK["W"]
    return oracle.trace_EX(W.A0, W.Bl, W.Br, W.Q, W.E, W.V[idx])


def _pick(W, count: int, seed: int):
    """A seeded sample of `count` grid rows: corners + centre + uniform when it is large enough to hold them
    (workloads' sample_indices), a plain seeded uniform choice otherwise."""
    import numpy as np
    if count >= len(W.corner_indices()) + 1:
        return W.sample_indices(count, seed=seed)[:count]
    rng = np.random.default_rng(7000 + seed)
    return np.sort(rng.choice(W.nv, size=min(count, W.nv), replace=False))


def oracle_rate(name: str, seconds: float, seed: int = 0):
    """Time the CPU oracle (as it stands) on a bounded sample: C single-threaded worker processes."""
    import multiprocessing as mp

    import workloads
    W = workloads.make(name)
    cores = os.cpu_count() or 1
    saved = {v: os.environ.get(v) for v in _THREAD_VARS}
    for v in _THREAD_VARS:
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_oracle_worker_init, initargs=(name,)) as pool:
        # first round: one v per core (warms the workers and sizes the sample).  When that round alone
        # is longer than the budget (c5: ~50 s per v), it IS the sample: no second pass.
        idx = _pick(W, cores, seed + 50)
        t = time.perf_counter()
        pool.map(_oracle_one, [int(i) for i in idx], chunksize=1)
        el = t1 = time.perf_counter() - t
        if t1 < seconds:
            t = time.perf_counter()  # the first round was cold: size the sample from a second, warm one
            pool.map(_oracle_one, [int(i) for i in _pick(W, cores, seed + 51)], chunksize=1)
            t1 = time.perf_counter() - t
            count = int(max(cores, min(W.nv, cores * max(1, int(seconds / max(t1, 1e-3))))))
            idx = _pick(W, count, seed)
            t = time.perf_counter()
            pool.map(_oracle_one, [int(i) for i in idx], chunksize=1)
            el = time.perf_counter() - t
    for v, val in saved.items():
        if val is None:
            os.environ.pop(v, None)
        else:
            os.environ[v] = val
    return len(idx) / el, cores, len(idx), el


# ------------------------------------------------------------------------------ helpers
def emit(obj):
    print(json.dumps(obj), flush=True)


def config_dict(W, args, world, extra=None):
    d = {"workload": W.name, "n": W.n, "k": W.k, "nv": W.nv, "grid": list(W.grid_shape),
         "seed": W.meta.get("seed"), "parallelism": f"v-grid sharded over {world} GPU(s)",
         "l2": "working set (Krylov bases, > 1 GB) exceeds the 126 MB L2; no flush needed"}
    if extra:
        d.update(extra)
    return d


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The reference arm: the CPU oracle (the paper's naive per-v Bartels-Stewart baseline) as it stands,
    on the host cores, one single-threaded worker per core; every step is a bounded seeded sample of the
    configuration's grid, sized so that the timed region of the whole run stays near BENCH_REF_SECONDS (240 s)
    whatever --steps is (c5: one v takes ~50 s on a busy box, so a step is 1-3 v)."""
    if rank != 0:
        return
    import multiprocessing as mp

    import workloads
    W = workloads.make(args.config)
    cores = os.cpu_count() or 1
    saved = {v: os.environ.get(v) for v in _THREAD_VARS}
    for v in _THREAD_VARS:
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    budget = float(os.environ.get("BENCH_REF_SECONDS", "240"))  # timed region of the whole --steps K run
    with ctx.Pool(cores, initializer=_oracle_worker_init, initargs=(args.config,)) as pool:
        # sizing round = first warm-up round: one v per core
        t = time.perf_counter()
        pool.map(_oracle_one, [int(i) for i in _pick(W, cores, 100)], chunksize=1)
        t1 = time.perf_counter() - t
        # further warm-up rounds (one v per core each), at most ~60 s of them
        for s_ in range(1, max(1, min(args.warmup, int(60.0 / max(t1, 1e-3))))):
            t = time.perf_counter()
            pool.map(_oracle_one, [int(i) for i in _pick(W, cores, 100 + s_)], chunksize=1)
            t1 = time.perf_counter() - t  # a warm round sizes the steps better than the cold first one
        # K steps inside `budget` seconds: rounds of one v per core that fit, dealt evenly to the steps
        # (at least one v per step).  All steps' samples go to the pool as ONE task list, so the cores
        # stay busy across step boundaries and only the last round can be ragged; value = v / wall.
        rounds = max(1, int(budget / max(t1, 1e-3)))
        per_step = int(max(1, min(W.nv, rounds * cores // max(args.steps, 1))))
        tasks = []
        for s_ in range(args.steps):
            tasks += [int(i) for i in _pick(W, per_step, 2 + s_)]
        t_all = time.perf_counter()
        pool.map(_oracle_one, tasks, chunksize=1)
        wall = time.perf_counter() - t_all
    for v, val in saved.items():
        if val is None:
            os.environ.pop(v, None)
        else:
            os.environ[v] = val
    value = len(tasks) / wall
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1),
          "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
          "data": "synthetic (seeded workloads.make)",
          "config": config_dict(W, args, world, {"sample_per_step": per_step}),
          "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                           "sample": f"{per_step} seeded grid points per step ({len(tasks)} in all, one task list "
                                     f"over {cores} single-threaded workers, {wall:.1f} s), blocked Bartels-Stewart "
                                     "per v, 1 BLAS thread"},
          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ------------------------------------------------------------------------------ our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import workloads
    from paper_2312_08201_b200 import Problem
    from paper_2312_08201_b200.sweep import Sweep

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    W = workloads.make(args.config)
    P = Problem(W.A0, W.Bl, W.Br, W.Q, W.E, profile=not args.no_profile, device=local, batch=args.batch, max_dim=args.max_dim,
                coarse=args.coarse, mixed=args.mixed,
                mixed_eta=args.mixed_eta)
    cost = P.cost_proxy(W.V)  # the engine's scheduling proxy: balances the strong-scaling shards
    emu = None
    if args.emulate_rank:
        er, en = (int(x) for x in args.emulate_rank.split("/"))
        emu = (er, en)
        from paper_2312_08201_b200.sweep import shard_indices
    sweep = Sweep(W.nv, rank, world, dev, scaling=args.scaling, cost=cost)
    if args.scaling == "weak":
        Vrank = workloads.rank_grid(W, rank, world)
        idx = np.arange(len(Vrank))
    else:
        Vrank = W.V
        idx = sweep.mine if emu is None else shard_indices(W.nv, emu[0], emu[1], cost=cost)
    nv_total = sweep.nv if emu is None else len(idx)
    setup_ms = P.info["setup_ms"]
    recycle_ms = None
    if args.recycle > 0:
        t = time.perf_counter()
        P.build_recycle(V=W.V, s=args.recycle)
        recycle_ms = 1e3 * (time.perf_counter() - t)
    Vd = torch.tensor(Vrank[idx], device=dev)

    if emu is not None:
        def step():
            tau = P.trace_batch(Vd)
            return tau, torch.argmin(tau)
    else:
        def step():
            return sweep.run(lambda rows: P.trace_batch(Vd))

    for _ in range(args.warmup):
        full, am = step()
    torch.cuda.synchronize()
    if recycle_ms is None and P.stats["recycle_build_ms"] > 0:  # automatic spaces, built during warm-up
        recycle_ms = P.stats["recycle_build_ms"]
    P.reset_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        full, am = step()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    st = P.stats
    value = nv_total * args.steps / (ms_max * 1e-3)
    argmin = int(am.item())

    # e2e: host buffers through the public API (H2D of V and D2H of traces inside the timed region)
    e2e = None
    if not args.no_e2e:
        Vh = np.ascontiguousarray(Vrank[idx])
        P.trace_batch(Vh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            tau_h = P.trace_batch(Vh)
        el = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e = {"value": nv_total * args.steps / float(el.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(Vh.nbytes), "d2h_bytes_per_step": int(len(idx) * (8 + 4 + 4 + 8))}

    avg_k1_ms = st["k1_ms"] / max(st["k1_launches"], 1)
    flops_per_launch = st["k1_flops"] / max(st["k1_launches"], 1)
    achieved = flops_per_launch / (avg_k1_ms * 1e-3) / 1e12 if avg_k1_ms > 0 else 0.0
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"k1_traffic_{args.config}.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get("bytes_per_launch")
    roof = {"bound": "tensor", "dtype": "f64", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "kernel": "k1_dgemm (Cauchy-fused T-apply GEMM, DMMA)",
            "peak_source": "measured DMMA mma.sync.m8n8k4.f64 microbench (profiles/r01_fp64_peaks.md); "
                           "MEASURED_PEAKS.json carries no FP64 figure",
            "avg_launch_ms": avg_k1_ms, "launches": st["k1_launches"],
            "k1_share_of_step": st["k1_ms"] / ms if ms > 0 else None}
    if P.mixed:
        # mixed precision: the dominant kernel is the tcgen05 3xTF32 GEMM of the Krylov
        # steps; its tensor work = 3 TF32 passes x 2 n^2 k^2 per ITER vector.  The timed region of each
        # launch (CUDA events on the engine stream) spans that kernel, its fused epilogue, and the exact
        # DMMA GEMM of the VERIFY vectors on the side stream (joined).
        mode = P.info["mixed_mode"]
        if mode == 3:  # 3xFP16 on tcgen05: the FP16 dense peak = the measured bf16 one (same rate)
            peak, psrc, burst = bf16_peak()
            dt = "f16 (3xFP16: hi/lo split with power-of-two scales, 3 passes, FP32 accumulation in TMEM)"
        else:
            peak, psrc = tf32_peak()
            burst = peak
            dt = "tf32 (3xTF32: hi/lo split, 3 passes, FP32 accumulation in TMEM)"
        it_vec = st["k1_vectors"] - st["k1_exact_vectors"]
        fl = 3.0 * 2.0 * W.n ** 2 * W.k ** 2 * it_vec
        a_tf = fl / (st["k1_ms"] * 1e-3) / 1e12 if st["k1_ms"] > 0 else 0.0
        tfile = os.path.join(ROOT, "profiles", f"umma_traffic_{args.config}.json")
        utraffic = json.load(open(tfile)).get("bytes_per_launch") if os.path.exists(tfile) else None
        roof = {"bound": "tensor", "dtype": dt,
                "achieved": a_tf, "peak": peak, "unit": "TFLOP/s", "frac": a_tf / peak, "traffic": utraffic,
                "kernel": "k1_umma_persistent (tcgen05.mma, TMA, TMEM; K1 epilogue fused)",
                "peak_source": psrc, "peak_burst": burst, "frac_of_burst": a_tf / burst,
                "avg_launch_ms": avg_k1_ms, "launches": st["k1_launches"],
                "k1_share_of_step": st["k1_ms"] / ms if ms > 0 else None,
                "work": "3 x 2 n^2 k^2 flops per ITER vector; VERIFY vectors (exact FP64, k1_dgemm on a side "
                        "stream inside the same timed region) not counted",
                "exact_fp64": {"kernel": "k1_dgemm (VERIFY applications)", "vectors": st["k1_exact_vectors"],
                               "vectors_total": st["k1_vectors"]}}
    # informational: K1 alone at full width (lyap_apply_C, outside the timed region, nothing else
    # running), the figure ncu reports per launch; roofline.achieved above is the timed-region average
    iso = None
    try:
        # one slot group's width (mixed precision runs one group over all slots)
        nvec = int(P.info["batch"]) if P.mixed else int(P.info["batch"] + 1) // 2
        Xt = torch.randn(nvec, W.k, P.info["npad"], dtype=torch.float64, device=dev)
        Xt[:, :, W.n:] = 0
        P.apply_C(Xt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.apply_C(Xt)
        e1.record()
        torch.cuda.synchronize()
        t_iso = e0.elapsed_time(e1) / 5 * 1e-3
        a_iso = 2.0 * W.n ** 2 * W.k ** 2 * nvec / t_iso / 1e12
        iso = {"vectors": nvec, "ms_per_apply": t_iso * 1e3, "achieved": a_iso, "frac": a_iso / FP64_PEAK_TFLOPS,
               "note": "whole K1 (prologue + GEMM + epilogue) alone at full width"}
    except Exception as exc:  # informational only
        iso = {"error": str(exc)}
    roof["isolated_k1"] = iso
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, cores, cnt, el = oracle_rate(args.config, args.cpu_seconds)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{cnt} of {W.nv} grid points (seeded sample) in {el:.1f} s, "
                         "blocked Bartels-Stewart per v, one process per core, 1 BLAS thread"}
    balance = None
    if args.scaling == "strong":
        from paper_2312_08201_b200.sweep import shard_balance
        balance = {str(N): round(shard_balance(W.nv, N, cost), 4) for N in (2, 4, 8)}
    if rank == 0:
        emit({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
              "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded workloads.make)",
              "config": config_dict(W, args, world, {"batch": P.info["batch"], "max_dim": P.info["max_dim"],
                                                     "nv_total": nv_total,
                                                     "setup_ms": setup_ms, "argmin_flat_index": argmin,
                                                     "recycle_s": args.recycle if args.recycle > 0 else ("auto" if recycle_ms else 0),
                                                     "recycle_build_ms": recycle_ms,
                                                     "applies_per_v": st["k1_vectors"] / (len(idx) * args.steps),
                                                     "exact_applies_per_v": st["k1_exact_vectors"] / (len(idx) * args.steps),
                                                     "mixed": P.mixed, "mixed_mode": P.info["mixed_mode"],
                                                     "shard_cost_max_over_mean": balance,
                                                     "coarse": P.info["coarse"],
                                                     "coarse_build_ms": P.info["coarse_build_ms"],
                                                     "emulated_rank": args.emulate_rank or None}),
              "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
              "gpu_launches": st["kernel_launches"]})
    P.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
