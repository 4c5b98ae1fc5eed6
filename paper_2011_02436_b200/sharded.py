"""Row-sharded training across ranks (one process per GPU).

The hot path shards naturally by rows: each rank builds H for its
contiguous block of rows and its local augmented Gram [H_p T_p]^T [H_p T_p]
((L+m) x (L+m): G_p and (H^T T)_p in one buffer); ONE all-reduce (sum) of its packed
lower triangle ((L+m)(L+m+1)/2 doubles: G and H^T T, half the bytes of the full
buffer); every rank then runs the identical pivoted-Cholesky + triangular solve, so
beta is bitwise identical on all ranks; training-accuracy hits are a local count
plus an all-reduce.

``fixed_order=True`` replaces the all-reduce by an all-gather of the packed partials
and a sum in rank order on every rank: the Gram then no longer depends on the
collective's internal reduction order, so exact ties between duplicated hidden
nodes (config 3) survive sharding.

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
        self._packed = None

    def pack(self, g):
        import torch

        n = g.shape[0]
        if self._packed is None or self._packed.numel() != n * (n + 1) // 2 or self._packed.device != g.device:
            self._packed = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=g.device)
        api.pack_lower_device(g, self._packed, ctx=self.ctx)
        return self._packed

    def unpack(self, packed, g) -> None:
        api.unpack_lower_device(packed, g, ctx=self.ctx)

    def sum_parts(self, parts, out) -> None:
        api.sum_parts_device(parts, out, ctx=self.ctx)

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


def _host_staged(t, group) -> bool:
    import torch.distributed as dist

    return t.is_cuda and dist.get_backend(group) != "nccl"


def exchange_gram(gaug, stages, group=None, fixed_order: bool = False) -> None:
    """The path's one exchange step, in place on gaug (square, symmetric): pack the lower triangle,
    all-reduce it (or all-gather + fixed-order sum), unpack to the summed symmetric Gram."""
    import torch
    import torch.distributed as dist

    packed = stages.pack(gaug)
    if _host_staged(packed, group):
        torch.cuda.synchronize(packed.device)  # host-staged backends (gloo) do not order against the stream
    if fixed_order:
        world = dist.get_world_size(group)
        parts = torch.empty((world, packed.numel()), dtype=packed.dtype, device=packed.device)
        dist.all_gather(list(parts.unbind(0)), packed, group=group)
        stages.sum_parts(parts, packed)
    else:
        dist.all_reduce(packed, group=group)
    stages.unpack(packed, gaug)


def train_sharded(x_local, t_local, params: api.ElmParams, strategy: api.SolverStrategy, n_total: int,
                  stages=None, group=None, hidden: Optional[api.HiddenLayer] = None, fixed_order: bool = False):
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
        exchange_gram(gaug, stages, group, fixed_order)  # the one exchange step of the path
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
                       stages: Optional[DeviceStages] = None, group=None, fixed_order: bool = False):
    """train() step of one rank on device-resident inputs (bench.py's timed step at N > 1): local
    augmented Gram, ONE all-reduce, replicated solve, hit-count all-reduce.  w, b are the
    replicated hidden layer as device tensors.  Returns (beta, SolveDiagnostics, order)."""
    import torch
    import torch.distributed as dist

    stages = stages or DeviceStages()
    gaug = stages.gram_aug(x_local, t_local, w, b)
    exchange_gram(gaug, stages, group, fixed_order)
    L, m = w.shape[1], t_local.shape[1]
    beta, diag, order = stages.solve_aug(gaug, L, m, n_total, strategy)
    hits = torch.tensor([stages.hits(x_local, t_local, w, b, beta)], dtype=torch.int64, device=gaug.device)
    if _host_staged(hits, group):
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
