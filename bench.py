#!/usr/bin/env python
"""Benchmark of the B200 RBP-ELM training hot path (BASELINE.json metric).

One "step" = one full train() with the rank strategy on the workload: H build (K1) ->
Gram/H^T T (K2) -> pivoted Cholesky (K3 + trailing SYRK) -> triangular solves (K4) ->
training-accuracy pass, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--scaling weak|strong]
                  [--impl ours|reference]

Default workload: BASELINE config 5 ("C5", d=256, L=8192, m=100), 500k rows per GPU -- the
largest single-GPU configuration (one shard of C5; the whole 4M-row C5 at 8 GPUs).  `--scaling
weak` (C5's default) keeps the rows per GPU fixed; `--scaling strong` (the C2/C4 default) keeps
the config's total row count and splits it over the ranks.  N > 1 runs under torchrun: each rank
builds the augmented Gram [H T]^T [H T] of its contiguous row shard, NCCL all-reduces its packed
lower triangle, every rank runs the replicated solve, hit counts are all-reduced.  Rank 0 prints
one JSON line.

`--impl reference` times the reference algorithm on the host CPU: the oracle restatement (the
reference itself cannot be built: no Eigen), all host threads, on a bounded sample of
the same workload (see reference_sample); that process never loads the product library.
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

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# name: (rows, d, L, m, default scaling).  rows are per GPU for weak scaling (C5: "H rows sharded
# 500k per GPU") and the job total for strong scaling (C2: N=50000, C4: N=100000).
CONFIGS = {
    "c1": (2000, 16, 200, 2, "strong"),
    "c2": (50000, 64, 1000, 10, "strong"),
    "c4_250": (100000, 128, 250, 10, "strong"),
    "c4_500": (100000, 128, 500, 10, "strong"),
    "c4_1000": (100000, 128, 1000, 10, "strong"),
    "c4_2000": (100000, 128, 2000, 10, "strong"),
    "c4_4000": (100000, 128, 4000, 10, "strong"),
    "c4_8000": (100000, 128, 8000, 10, "strong"),
    "c5": (500000, 256, 8192, 100, "weak"),
}
DEFAULT_CONFIG = "c5"
SEED_X, SEED_TEACHER, SEED_W = 1002, 2002, 3002
METRIC = ("ELM train FP64 TFLOP/s (alg. flops of H build + Gram + pivoted Cholesky + solves + accuracy "
          "/ train time)")
DATA = "synthetic (seeded mt19937_64 generators, SURVEY 8(d)); random-init W, b from init_hidden"


def alg_flops(n, d, L, m):
    """2NdL + N L(L+1) + 2NLm + L^3/3 + 2L^2 m + 2NLm."""
    return 2 * n * d * L + n * L * (L + 1) + 2 * n * L * m + L ** 3 / 3 + 2 * L * L * m + 2 * n * L * m


def row_flops(d, L, m):
    """Per-row part of alg_flops (hidden build, Gram, H^T T, accuracy pass)."""
    return 2 * d * L + L * (L + 1) + 4 * L * m


def workload(args, world):
    """(config dict, rows of this rank, total rows, d, L, m).  The dict is printed identically by both
    arms (the driver compares them)."""
    rows, d, L, m, default_scaling = CONFIGS[args.config]
    scaling = args.scaling or default_scaling
    n_total = rows * world if scaling == "weak" else rows
    n_rank = n_total // world  # rank r owns rows [r * n_rank, (r + 1) * n_rank) (+ remainder on the last)
    desc = (f"{args.config}: N_total={n_total} ({n_total // world}/GPU) d={d} L={L} m={m}, rank strategy "
            f"(default tol), full train() incl. training-accuracy pass")
    cfg = {"workload": desc, "N_total": n_total, "d": d, "L": L, "m": m, "scaling": scaling,
           "l2": "inputs > L2 (126 MB) and a 256 MB L2 flush write between timed steps, outside the events",
           "parallelism": f"row-sharded dp{world} (NCCL all-reduce of the packed Gram)" if world > 1 else "single GPU"}
    return cfg, n_rank, n_total, d, L, m


def fp64_peak():
    """Measured FP64 GEMM peak (cuBLAS DGEMM 8192^3, best of 10) -- MEASURED_PEAKS.json has no FP64 entry."""
    path = os.path.join(HERE, "profiles", "fp64_peak_r01.json")
    try:
        with open(path) as f:
            return float(json.load(f)["cublas_dgemm_8192_tflops"]), "measured cuBLAS DGEMM 8192^3 (profiles/fp64_peak_r01.json)"
    except Exception:
        return 37.0, "fallback datasheet-class FP64 figure"


def int8_peak():
    """INT8 dense tensor peaks (sustained, burst): twice the measured bf16 cuBLAS rates of MEASURED_PEAKS.json
    (the int8 MMA rate is twice bf16's; nominal 4.5 POP/s).  The Gram runs ~70 % of a long step at the
    power cap, so the sustained figure is its roofline denominator (B200_PROFILING: sustained for a kernel
    timed inside a long step); the burst one is reported beside it."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        burst = 2.0 * float(mp["bf16_tflops"])
        sus = 2.0 * float(mp.get("bf16_tflops_sustained", mp["bf16_tflops"]))
        return sus, burst, ("2 x MEASURED_PEAKS.json bf16_tflops_sustained (int8 MMA rate = 2x bf16; "
                            "the Gram runs inside a long step at the power cap)")
    except Exception:
        return 2.0 * 1590.0, 2.0 * 1590.0, "2 x fallback bf16 1.59 PFLOP/s (B200_PROFILING.md)"


def hbm_peak():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6518.0, "fallback (round-1 MEASURED_PEAKS.json figure)"


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
            self._stop.wait(0.1)

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


# ---------------------------------------------------------------------------------------------
# CPU legs (oracle restatement only; this code path never imports the product package)
# ---------------------------------------------------------------------------------------------
def reference_sample(n_total, d, L, m, threads, rows=None):
    """Time the oracle's train(rank) on a bounded sample of the workload and extrapolate to N_total rows.

    Phases that are linear in the row count (hidden build, Gram + H^T T, accuracy pass) run on the
    first R rows of the workload (R sized for ~1.5e11 flops of row work, all rows when the whole
    workload is that small); the row-count-independent phases (pivoted Cholesky of the L x L Gram,
    triangular solves) run at full L.  time = row phases * N_total / R + factor + solve.
    Returns (TFLOP/s, seconds, R, phases)."""
    import oracle

    if rows is None:
        rows = int(1.5e11 // row_flops(d, L, m))
        rows = max(256, (rows // 256) * 256)
    rows = min(rows, n_total)
    x, t = oracle.synth_classification(rows, d, m, SEED_X, SEED_TEACHER)
    oracle.set_threads(threads)
    ph = oracle.train_phase_times(d, L, m, SEED_W, x, t)
    per_rows = ph["hidden"] + ph["gram"] + ph["accuracy"]
    sec = per_rows * (n_total / rows) + ph["factor"] + ph["solve"]
    return alg_flops(n_total, d, L, m) / sec / 1e12, sec, rows, ph


def sample_text(cfg_name, rows, n_total, L, threads, ph):
    how = ("whole workload" if rows >= n_total else
           f"hidden build, Gram + H^T T and accuracy pass timed on the first {rows} of {n_total} rows and scaled "
           f"linearly to N_total; pivoted Cholesky + triangular solves timed at full L={L}"
           + (" on the sample Gram + 1e-2 max(diag) I (full rank)" if rows < L else ""))
    return (f"oracle restatement of train(rank), bitwise equal to the reference's own sources built on an Eigen stand-in "
            f"(oracle/_ref: scalar, single-threaded, so the faster port is the one timed; real Eigen is absent), "
            f"{threads} host threads, "
            f"{cfg_name}: {how}; phases {', '.join(f'{k} {v:.2f}s' for k, v in ph.items() if k != 'rank')}")


def reference_arm(args, rank, world):
    if rank != 0:
        return
    cfg, _, n_total, d, L, m = workload(args, world)
    threads = os.cpu_count() or 1
    samples = []
    for i in range(args.warmup + args.steps):
        v, sec, rows, ph = reference_sample(n_total, d, L, m, threads)
        if i >= args.warmup:
            samples.append((v, sec, rows, ph))
    value = statistics.mean(s[0] for s in samples)
    sec = statistics.mean(s[1] for s in samples)
    rows, ph = samples[-1][2], samples[-1][3]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "higher_is_better": True,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": DATA, "config": cfg,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                         "sample": sample_text(args.config, rows, n_total, L, threads, ph)},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2011_02436_b200 as rb
    from paper_2011_02436_b200 import sharded

    cfg, n, N_total, d, L, m = workload(args, world)
    row0 = rank * n
    if rank == world - 1:
        n = N_total - row0  # the remainder rows go to the last rank

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
    xh, th = rb.synth_classification(n, d, m, SEED_X, SEED_TEACHER, row0=row0)
    X = torch.from_numpy(xh).to(dev)
    T = torch.from_numpy(th).to(dev)
    params = rb.ElmParams(d, L, m, SEED_W)
    hidden = rb.init_hidden(params)
    W = torch.from_numpy(hidden.weights).to(dev)
    B = torch.from_numpy(hidden.biases.reshape(-1)).to(dev)
    ctx = rb.context(local_dev)
    strat = rb.SolverStrategy.rank_based()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    stages = sharded.DeviceStages(ctx) if world > 1 else None

    def step():
        if world == 1:
            beta, diag, _ = rb.train_device(X, T, params, strat, hidden=hidden, ctx=ctx)
            return diag
        # row shard -> augmented Gram -> ONE all-reduce of its packed lower triangle -> replicated solve
        beta, diag, _ = sharded.train_shard_device(X, T, W, B, params, strat, N_total, stages=stages)
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
    prof = {k: ctx.profile(k) for k in ("hidden_kernel", "oz_colmax", "oz_slice", "oz_gram_kernel", "syrk_kernel",
                                        "syrk_finish", "panel_kernel", "syrk_trailing", "trsm_pair_kernel",
                                        "scores_kernel")}
    ctx.set_profiling(False)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_step = float(t_max.item()) / args.steps
    flops = alg_flops(N_total, d, L, m)
    value = flops / (ms_step * 1e-3) / 1e12

    # ---- e2e: the reference-facing call with HOST buffers, host<->device copies inside the timed region
    xp = torch.empty((n, d), dtype=torch.float64).pin_memory()
    tp = torch.empty((n, m), dtype=torch.float64).pin_memory()
    xp.copy_(torch.from_numpy(xh))
    tp.copy_(torch.from_numpy(th))
    if world > 1:
        def e2e_step():  # pinned host shard -> device -> sharded train -> beta back to the host
            xd = xp.to(dev, non_blocking=True)
            td = tp.to(dev, non_blocking=True)
            beta, dg, _, _ = sharded.train_sharded(xd, td, params, strat, N_total, stages=stages, hidden=hidden)
            return beta.cpu()
        api = "sharded.train_sharded (Python API, pinned host shard per rank; max over ranks)"
    else:
        xpn, tpn = xp.numpy(), tp.numpy()
        ctx.set_stream(0)

        def e2e_step():
            return rb.train(params, xpn, tpn, strat, ctx=ctx)
        api = "rbpg_train (C ABI, host buffers)"
    e2e_step()
    t_e = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        t_e.append(float(te.item()))
    e2e_s = statistics.median(t_e)
    e2e = {"value": flops / e2e_s / 1e12, "unit": "TFLOP/s", "seconds": e2e_s,
           "h2d_bytes_per_step": int(n * d * 8 + n * m * 8), "d2h_bytes_per_step": int(L * m * 8), "api": api}

    # ---- batched prediction (elm.cpp:282-284) on this rank's rows: device-resident X, labels out
    ctx.set_stream(rb.api._torch_stream(dev))
    beta_d, _, _ = rb.train_device(X, T, params, strat, hidden=hidden, ctx=ctx)
    pr = min(n, 200000)
    Xp = X[:pr]
    labels = torch.empty(pr, dtype=torch.int32, device=dev)
    rb.predict_labels_device(Xp, W, B, beta_d, labels, ctx=ctx)
    torch.cuda.synchronize()
    pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a, b in pe:
        flush.zero_()
        a.record(stream)
        rb.predict_labels_device(Xp, W, B, beta_d, labels, ctx=ctx)
        b.record(stream)
    torch.cuda.synchronize()
    pms = statistics.median(a.elapsed_time(b) for a, b in pe)
    pflops = 2 * pr * L * (d + m)
    pred = {"rows": pr, "ms": pms, "TFLOP/s": pflops / (pms * 1e-3) / 1e12,
            "frac_fp64_peak": pflops / (pms * 1e-3) / 1e12 / fp64_peak()[0],
            "alg_flops": pflops, "hbm_bytes": pr * d * 8 + pr * 4,
            "kernel": ("INT8 path (m > 48): K1i hidden build of row chunks + digit planes + K6i scores with the arg-max "
                       "epilogue; TFLOP/s are FP64-equivalent" if m > 48 else
                       "predict_kernel (K6b: fused sigma(XW+b) beta + arg-max labels on DMMA; H never stored)")}

    if rank == 0:
        peak, peak_src = fp64_peak()
        n_local = n
        gram_flops = n_local * (L + m) * (L + m + 1)  # augmented lower-triangle Gram of [H T] (K2)
        # the Gram runs on the INT8 tensor cores (k_ozaki.cu): 28 exact int8 products of the digit
        # planes per element; roofline = those int8 ops over the kernel's time against the INT8 dense
        # peak, taken as twice the measured bf16 cuBLAS rate (the int8 MMA rate is twice bf16's)
        oz_ms, oz_n = prof["oz_gram_kernel"]
        int8_ops = 28 * gram_flops
        i8_peak, i8_burst, i8_src = int8_peak()
        achieved = int8_ops / (oz_ms / oz_n * 1e-3) / 1e12 if oz_n else None
        gram_ms_per = sum(prof[k][0] for k in ("oz_colmax", "oz_slice", "oz_gram_kernel", "syrk_finish")) / max(oz_n, 1)
        fp64_equiv = gram_flops / (gram_ms_per * 1e-3) / 1e12 if oz_n else None
        # algorithmic bytes of one Gram launch: the 7 digit planes read once, the packed partial tiles
        # (2 accumulator groups x int32-safe row splits) written once
        nbI = (L + m + 127) // 128
        Mpad = (nbI + 1) // 2 * 256
        Npad = (n_local + 63) // 64 * 64
        splits = max(1, (n_local + 16383) // 16384)
        alg_bytes = 7 * Npad * Mpad + 2 * splits * (nbI * (nbI + 1) // 2) * 16384 * 8
        traffic = None
        tpath = os.path.join(HERE, "profiles", "traffic_r02.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(args.config, {}).get("gram")
            except Exception:
                traffic = None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            v, sec, rows, ph = reference_sample(N_total, d, L, m, threads)
            cpu = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                   "sample": sample_text(args.config, rows, N_total, L, threads, ph)}
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": cfg["scaling"],
            "vs_baseline": None, "dtype": "f64", "data": DATA, "config": cfg,
            "arithmetic": ("f64 throughout; the Gram's products are exact int8 tensor-core products of 7 digit planes "
                           "per fp64 value (54-bit integers per column scale), combined in fp64: max error 1.1e-16 "
                           "of sqrt(G_aa G_bb) vs an exact reference (a sequential fp64 sum: 5e-15), tests/test_ozaki_gpu.py"),
            "train_ms": ms_step, "rank": diag.rank, "training_accuracy": diag.training_accuracy,
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
            "roofline": {"kernel": "K2i oz_gram_kernel: Gram of [H T] on the INT8 tensor cores (tcgen05.mma "
                                   "kind::i8, 7 exact digit planes, 28 products, fp64 combination)",
                         "bound": "tensor", "achieved": achieved, "peak": i8_peak, "unit": "TOP/s (int8)",
                         "frac": (achieved / i8_peak) if achieved else None, "traffic": traffic,
                         "traffic_source": "profiles/traffic_r02.json (ncu --set full, dram read + write per launch)",
                         "alg_bytes_per_launch": alg_bytes,
                         "peak_source": i8_src, "peak_burst": i8_burst,
                         "frac_of_burst": (achieved / i8_burst) if achieved else None,
                         "alg_ops_per_launch": int8_ops, "launches": oz_n,
                         "fp64_equivalent": {"what": "whole Gram stage (column scan + digit planes + int8 products + "
                                                     "split reduction) as FP64 Gram flops L'(L'+1)N / time, L'=L+m",
                                             "TFLOP/s": fp64_equiv, "frac_of_dgemm_peak": (fp64_equiv / peak) if fp64_equiv else None,
                                             "dgemm_peak": peak, "dgemm_peak_source": peak_src}},
            "predict": pred,
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
