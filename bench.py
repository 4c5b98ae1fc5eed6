#!/usr/bin/env python
"""Benchmark of the B200 RBP-ELM training hot path (BASELINE.json metric).

One "step" = one full train() with the rank strategy on the workload:
H build (K1) -> Gram/H^T T (K2) -> pivoted Cholesky (K3 + trailing SYRK) ->
triangular solves (K4) -> training-accuracy pass, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

N > 1 runs under torchrun: rows are sharded (weak scaling, config rows per GPU),
each rank builds its local Gram/H^T T, NCCL all-reduces them, every rank runs the
replicated solve, hit counts are all-reduced.  Rank 0 prints one JSON line.

`--impl reference` times the reference algorithm on the host CPU (the oracle
restatement, all host threads; the reference itself cannot be built here -- no
Eigen) on a bounded row sample of the same workload.
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

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# (N rows per GPU, d, L, m) -- BASELINE.json configs
CONFIGS = {
    "c1": (2000, 16, 200, 2),
    "c2": (50000, 64, 1000, 10),
    "c4_250": (100000, 128, 250, 10),
    "c4_500": (100000, 128, 500, 10),
    "c4_1000": (100000, 128, 1000, 10),
    "c4_2000": (100000, 128, 2000, 10),
    "c4_4000": (100000, 128, 4000, 10),
    "c4_8000": (100000, 128, 8000, 10),
    "c5": (500000, 256, 8192, 100),
}
SEED_X, SEED_TEACHER, SEED_W = 1002, 2002, 3002


def alg_flops(n, d, L, m):
    """2NdL + N L(L+1) + 2NLm + L^3/3 + 2L^2 m + 2NLm."""
    return 2 * n * d * L + n * L * (L + 1) + 2 * n * L * m + L ** 3 / 3 + 2 * L * L * m + 2 * n * L * m


def fp64_peak():
    """Measured FP64 GEMM peak (cuBLAS DGEMM 8192^3, best of 10) -- MEASURED_PEAKS.json has no FP64 entry."""
    path = os.path.join(HERE, "profiles", "fp64_peak_r01.json")
    try:
        with open(path) as f:
            return float(json.load(f)["cublas_dgemm_8192_tflops"]), "measured cuBLAS DGEMM 8192^3 (profiles/fp64_peak_r01.json)"
    except Exception:
        return 37.0, "fallback datasheet-class FP64 figure"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_oracle_sample(n, d, L, m, threads, rows):
    """Time the oracle's train() on the first `rows` rows of the workload (TFLOP/s)."""
    import oracle
    import paper_2011_02436_b200 as rb  # data generator only

    rows = min(rows, n)
    x, t = rb.synth_classification(rows, d, m, SEED_X, SEED_TEACHER)
    oracle.set_threads(threads)
    t0 = time.perf_counter()
    oracle.train(d, L, m, SEED_W, x, t, "rank")
    dt = time.perf_counter() - t0
    return alg_flops(rows, d, L, m) / dt / 1e12, dt


def reference_arm(args, n, d, L, m, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rows = int(os.environ.get("RBPG_REF_ROWS", str(n)))
    samples = []
    for i in range(args.warmup + args.steps):
        v, dt = cpu_oracle_sample(n, d, L, m, threads, rows)
        if i >= args.warmup:
            samples.append((v, dt))
    value = statistics.mean(v for v, _ in samples)
    sec = statistics.mean(dt for _, dt in samples)
    line = {
        "impl": "reference",
        "metric": "ELM train FP64 TFLOP/s (alg. flops of H build + Gram + pivoted Cholesky + solves + accuracy / train time)",
        "value": value, "unit": "TFLOP/s", "higher_is_better": True, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded mt19937_64, SURVEY 8(d))",
        "config": {"workload": f"{args.config}: N={n}/GPU d={d} L={L} m={m}, rank strategy", "sample_rows": min(rows, n)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                         "sample": f"oracle restatement train() on the first {min(rows, n)} rows of {args.config} "
                                   f"(L={L}, d={d}, m={m}), {threads} threads; reference not buildable (no Eigen)"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n, d, L, m = CONFIGS[args.config]

    if args.impl == "reference":
        reference_arm(args, n, d, L, m, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2011_02436_b200 as rb

    # RBPG_DIST_BACKEND=gloo + more ranks than GPUs: a functional check of the sharded orchestration
    # on one GPU (host-staged all-reduce; not a scaling measurement)
    backend = os.environ.get("RBPG_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    # ---- inputs: this rank's contiguous row shard of the global matrix, resident in HBM
    xh, th = rb.synth_classification(n, d, m, SEED_X, SEED_TEACHER, row0=rank * n)
    X = torch.from_numpy(xh).to(dev)
    T = torch.from_numpy(th).to(dev)
    params = rb.ElmParams(d, L, m, SEED_W)
    hidden = rb.init_hidden(params)
    W = torch.from_numpy(hidden.weights).to(dev)
    B = torch.from_numpy(hidden.biases.reshape(-1)).to(dev)
    ctx = rb.context(local_dev)
    strat = rb.SolverStrategy.rank_based()
    N_total = n * world
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    Gaug = torch.empty((L + m, L + m), dtype=torch.float64, device=dev)

    def step():
        if world == 1:
            beta, diag, _ = rb.train_device(X, T, params, strat, hidden=hidden, ctx=ctx)
            return diag
        # row shard -> augmented Gram [H T]^T [H T] -> ONE all-reduce -> replicated solve
        rb.gram_stage_device_aug(X, T, W, B, Gaug, ctx=ctx)
        if backend != "nccl":
            torch.cuda.synchronize()  # host-staged backends do not order against the stream
        dist.all_reduce(Gaug)
        beta, diag = rb.solve_stage_device_aug(Gaug, L, m, N_total, strat, ctx=ctx)
        hits = torch.tensor([rb.accuracy_stage_device(X, T, W, B, beta, ctx=ctx)], dtype=torch.int64, device=dev)
        if backend != "nccl":
            torch.cuda.synchronize()
        dist.all_reduce(hits)
        diag.training_accuracy = hits.item() / N_total
        return diag

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count
    with ClockSampler(local_dev) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            diag = step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = ctx.launch_count - launches0
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    # per-kernel breakdown from a separate pass with per-launch events (events between launches
    # would serialise the programmatic dependent launches of the timed steps)
    ctx.set_profiling(True)
    for i in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    syrk_ms, syrk_n = ctx.profile("syrk_kernel")
    hid_ms, hid_n = ctx.profile("hidden_kernel")
    panel_ms, panel_n = ctx.profile("panel_kernel")
    trail_ms, trail_n = ctx.profile("syrk_trailing")
    trsm_ms, trsm_n = ctx.profile("trsm_pair_kernel")
    ctx.set_profiling(False)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    ms_step = ms_max / args.steps
    flops = alg_flops(N_total, d, L, m)
    value = flops / (ms_step * 1e-3) / 1e12

    # ---- e2e: the reference-facing C-ABI call with host (pinned) buffers, copies inside the timed region
    e2e = None
    if world > 1:
        # the sharded train() through the Python API from this rank's pinned host shard: H2D of the
        # shard, augmented Gram, all-reduce, replicated solve, hit-count all-reduce, beta back to host
        from paper_2011_02436_b200 import sharded

        xp = torch.empty((n, d), dtype=torch.float64).pin_memory()
        tp = torch.empty((n, m), dtype=torch.float64).pin_memory()
        xp.copy_(torch.from_numpy(xh))
        tp.copy_(torch.from_numpy(th))
        stages = sharded.DeviceStages(ctx)

        def e2e_step():
            xd = xp.to(dev, non_blocking=True)
            td = tp.to(dev, non_blocking=True)
            beta, dg, _, _ = sharded.train_sharded(xd, td, params, strat, N_total, stages=stages, hidden=hidden)
            return beta.cpu()

        e2e_step()
        t_e = []
        for _ in range(max(3, args.steps)):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            t_e.append(float(te.item()))
        e2e_s = statistics.median(t_e)
        e2e = {"value": flops / e2e_s / 1e12, "unit": "TFLOP/s", "seconds": e2e_s,
               "h2d_bytes_per_step": int(n * d * 8 + n * m * 8), "d2h_bytes_per_step": int(L * m * 8),
               "api": "sharded.train_sharded (Python API, pinned host shard per rank; max over ranks)"}
    if world == 1:
        xp = torch.empty((n, d), dtype=torch.float64).pin_memory()
        tp = torch.empty((n, m), dtype=torch.float64).pin_memory()
        xp.copy_(torch.from_numpy(xh))
        tp.copy_(torch.from_numpy(th))
        xpn, tpn = xp.numpy(), tp.numpy()
        ctx.set_stream(0)
        rb.train(params, xpn, tpn, strat, ctx=ctx)  # warm
        t_e = []
        for _ in range(max(3, args.steps)):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            model, dg = rb.train(params, xpn, tpn, strat, ctx=ctx)
            t_e.append(time.perf_counter() - t0)
        e2e_s = statistics.median(t_e)
        e2e = {"value": flops / e2e_s / 1e12, "unit": "TFLOP/s", "seconds": e2e_s,
               "h2d_bytes_per_step": int(n * d * 8 + n * m * 8),
               "d2h_bytes_per_step": int(L * m * 8),  # beta (W, b are generated on the host)
               "api": "rbpg_train (C ABI, host buffers)"}

    if rank == 0:
        peak, peak_src = fp64_peak()
        syrk_flops = N_total // world * L * (L + 1) + 2 * (N_total // world) * L * m
        syrk_per_launch_ms = syrk_ms / max(syrk_n, 1)
        achieved = syrk_flops / (syrk_per_launch_ms * 1e-3) / 1e12 if syrk_n else None
        traffic = None
        tpath = os.path.join(HERE, "profiles", "traffic_r01.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(args.config, {}).get("syrk_kernel")
            except Exception:
                traffic = None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            rows = int(os.environ.get("RBPG_CPU_ROWS", str(n)))
            v, dt = cpu_oracle_sample(n, d, L, m, 1, rows)
            cpu = {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "port",
                   "sample": f"oracle restatement train() (single thread, as the reference build) on the first "
                             f"{min(rows, n)} rows of {args.config} (L={L}, d={d}, m={m}); {dt:.1f} s; host has "
                             f"{os.cpu_count()} cores"}
        line = {
            "metric": "ELM train FP64 TFLOP/s (alg. flops of H build + Gram + pivoted Cholesky + solves + accuracy / train time)",
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mt19937_64 generators, SURVEY 8(d)); random-init W, b from init_hidden",
            "config": {"workload": f"{args.config}: N={n}/GPU (N_total={N_total}) d={d} L={L} m={m}, rank strategy, "
                                   f"full train() incl. accuracy pass",
                       "l2": "flushed between timed steps (256 MB write outside the events)",
                       "parallelism": f"row-sharded dp{world}" if world > 1 else "single GPU"},
            "train_ms": ms_step, "rank": diag.rank, "training_accuracy": diag.training_accuracy,
            "kernel_ms_per_step": {"hidden_kernel": hid_ms / args.steps, "syrk_kernel": syrk_ms / args.steps,
                                   "panel_kernel": panel_ms / args.steps, "syrk_trailing": trail_ms / args.steps,
                                   "trsm_pair_kernel": trsm_ms / args.steps},
            "roofline": {"kernel": "syrk_kernel (K2 Gram H^T H + H^T T, DMMA)", "bound": "tensor",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "peak_source": peak_src,
                         "alg_flops_per_launch": syrk_flops, "launches": syrk_n},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
