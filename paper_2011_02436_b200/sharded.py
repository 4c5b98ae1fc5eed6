"""Row-sharded training across ranks (one process per GPU).

The hot path shards naturally by rows: each rank builds H for its
contiguous block of rows and its local augmented Gram [H_p T_p]^T [H_p T_p]
((L+m) x (L+m): G_p and (H^T T)_p in one buffer); ONE all-reduce (sum); every
rank then runs the identical pivoted-Cholesky + triangular solve, so beta is
bitwise identical on all ranks; training-accuracy hits are a local count plus an
all-reduce.

``train_sharded`` is the orchestration; the per-rank numerical stages are a
pluggable object.  ``DeviceStages`` (the product) runs them through the C ABI on
the rank's GPU and the all-reduce goes over NCCL/NVLink.  The default tolerance
uses the GLOBAL row count (reference linalg.cpp:171).
"""
from __future__ import annotations

from typing import Optional, Tuple

from . import api


def shard_rows(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous row block of `rank`: (first row, row count); the first n_total % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_total, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


class DeviceStages:
    """Per-rank stages on the local GPU (sm_100a kernels through the C ABI)."""

    def __init__(self, ctx: Optional[api.Context] = None):
        self.ctx = ctx

    def gram_aug(self, x, t, w, b):
        import torch

        M = w.shape[1] + t.shape[1]
        g = torch.empty((M, M), dtype=torch.float64, device=x.device)
        api.gram_stage_device_aug(x, t, w, b, g, keep_h=True, ctx=self.ctx)
        return g

    def solve_aug(self, gaug, L: int, m: int, n_total: int, strategy: api.SolverStrategy):
        return api.solve_stage_device_aug(gaug, L, m, n_total, strategy, ctx=self.ctx, return_order=True)

    def hits(self, x, t, w, b, beta) -> int:
        return api.accuracy_stage_device(x, t, w, b, beta, ctx=self.ctx)

    def as_tensor(self, x, like):
        import torch

        return torch.as_tensor(x, dtype=torch.float64, device=like.device)

    def gram_of(self, h):
        import torch

        g = torch.empty((h.shape[1], h.shape[1]), dtype=torch.float64, device=h.device)
        api.gram_device(h, g, ctx=self.ctx)
        return g

    def pinv_block(self, g, h, n_total: int, tol: float):
        return api.pseudo_inverse_stage_device(g, h, n_total, tol, ctx=self.ctx)


def train_sharded(x_local, t_local, params: api.ElmParams, strategy: api.SolverStrategy, n_total: int,
                  stages=None, group=None, hidden: Optional[api.HiddenLayer] = None):
    """Row-sharded train(): returns (beta, SolveDiagnostics, HiddenLayer, order).

    x_local / t_local are this rank's contiguous row block (``shard_rows``) as tensors on the
    rank's device; `stages` provides gram/solve/hits (DeviceStages by default).
    """
    import torch
    import torch.distributed as dist

    stages = stages or DeviceStages()
    hidden = hidden or api.init_hidden(params)  # identical on every rank (seeded mt19937_64)
    w = stages.as_tensor(hidden.weights, x_local)
    b = stages.as_tensor(hidden.biases.reshape(-1), x_local)
    gaug = stages.gram_aug(x_local, t_local, w, b)
    distributed = dist.is_available() and dist.is_initialized()
    if distributed:
        if gaug.is_cuda and dist.get_backend(group) != "nccl":
            torch.cuda.synchronize(gaug.device)  # host-staged backends (gloo) do not order against the stream
        dist.all_reduce(gaug, group=group)  # the one exchange step of the path
    L, m = w.shape[1], t_local.shape[1]
    beta, diag, order = stages.solve_aug(gaug, L, m, n_total, strategy)
    hits = torch.tensor([stages.hits(x_local, t_local, w, b, beta)], dtype=torch.int64, device=gaug.device)
    if distributed:
        if hits.is_cuda and dist.get_backend(group) != "nccl":
            torch.cuda.synchronize(hits.device)
        dist.all_reduce(hits, group=group)
    diag.training_accuracy = float(hits.item()) / float(n_total)
    return beta, diag, hidden, order


def train_shard_device(x_local, t_local, w, b, params: api.ElmParams, strategy: api.SolverStrategy, n_total: int,
                       stages: Optional[DeviceStages] = None, group=None):
    """train() step of one rank on device-resident inputs (bench.py's timed step at N > 1): local
    augmented Gram, ONE all-reduce, replicated solve, hit-count all-reduce.  w, b are the
    replicated hidden layer as device tensors.  Returns (beta, SolveDiagnostics, order)."""
    import torch
    import torch.distributed as dist

    stages = stages or DeviceStages()
    gaug = stages.gram_aug(x_local, t_local, w, b)
    if dist.get_backend(group) != "nccl":
        torch.cuda.synchronize(gaug.device)
    dist.all_reduce(gaug, group=group)
    L, m = w.shape[1], t_local.shape[1]
    beta, diag, order = stages.solve_aug(gaug, L, m, n_total, strategy)
    hits = torch.tensor([stages.hits(x_local, t_local, w, b, beta)], dtype=torch.int64, device=gaug.device)
    if dist.get_backend(group) != "nccl":
        torch.cuda.synchronize(hits.device)
    dist.all_reduce(hits, group=group)
    diag.training_accuracy = float(hits.item()) / float(n_total)
    return beta, diag, order


def pseudo_inverse_sharded(h_local, n_total: int, tol: float = 0.0, stages=None, group=None):
    """Row-sharded rank-path pseudo-inverse: each rank holds a contiguous
    row block H_p of H; one all-reduce of the local Grams H_p^T H_p, then every rank factors the
    same G and writes its own column block H^+[:, rows of p] = P (F F^T)^-1 P^T H_p^T with no
    further exchange.  Returns (block (L x n_local), order, rank)."""
    import torch.distributed as dist

    stages = stages or DeviceStages()
    g = stages.gram_of(h_local)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(g, group=group)
    return stages.pinv_block(g, h_local, n_total, tol)
