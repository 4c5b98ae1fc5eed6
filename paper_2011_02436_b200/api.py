"""Python mirror of the reference's train/predict API for the B200 hot path.

Names, argument meaning and error behaviour follow /root/reference/proj/include/
rbpelm/{matrix,linalg,elm}.hpp, so the parity tests read like the reference's
own doctest suites.  Matrices are numpy float64 arrays (row-major, as the
reference's DenseMatrix).  Every numerical call goes through the C ABI of
librbpelm_b200.so to the sm_100a kernels; there is no CPU fallback.

Device-resident entry points (``train_device`` and the three stage functions)
take torch CUDA tensors and are what bench.py and the row-sharded multi-GPU
driver use.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native
from ._native import rbpg_diagnostics, rbpg_status, rbpg_strategy

# ---------------------------------------------------------------------------
# exceptions (matrix.hpp:11-14, linalg.hpp:15-20, elm.hpp:67-72)
# ---------------------------------------------------------------------------


class ShapeError(ValueError):
    """Incompatible operand shapes (rbpelm::ShapeError, a std::invalid_argument)."""


class SingularMatrix(RuntimeError):
    def __init__(self, pivot_index: int, pivot_value: float, message: str = ""):
        super().__init__(message or f"non-positive pivot {pivot_value} at index {pivot_index}")
        self.pivot_index = int(pivot_index)
        self.pivot_value = float(pivot_value)


class SingularSplit(RuntimeError):
    A = 0
    D = 1

    def __init__(self, which: int, message: str = ""):
        super().__init__(message or f"singular {'A' if which == 0 else 'D'} block after ridge retry")
        self.which = int(which)


class DeviceError(RuntimeError):
    pass


class NotSupportedError(RuntimeError):
    pass


def _raise(st: rbpg_status) -> None:
    code = st.code
    if code == 0:
        return
    msg = st.message.decode(errors="replace")
    if code == 1:
        raise ShapeError(msg)
    if code == 2:
        raise ValueError(msg)  # std::invalid_argument
    if code == 3:
        raise SingularMatrix(st.pivot_index, st.pivot_value, msg)
    if code == 4:
        raise SingularSplit(st.block, msg)
    if code == 6:
        raise DeviceError(msg)
    if code == 7:
        raise NotSupportedError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------------------
# types (elm.hpp:13-63, linalg.hpp:25-29, 77-80)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SolverStrategy:
    kind: str = "direct"  # "direct" | "df" | "rank"
    split_index: int = 0
    rank_tol: float = 0.0

    @staticmethod
    def direct() -> "SolverStrategy":
        return SolverStrategy("direct", 0, 0.0)

    @staticmethod
    def df_split(split: int) -> "SolverStrategy":
        return SolverStrategy("df", int(split), 0.0)

    @staticmethod
    def rank_based(tol: float = 0.0) -> "SolverStrategy":
        return SolverStrategy("rank", 0, float(tol))

    def describe(self) -> str:  # elm.cpp:53-67
        if self.kind == "direct":
            return "direct"
        if self.kind == "df":
            return f"df:{self.split_index}"
        return "rank" if self.rank_tol <= 0.0 else f"rank:{self.rank_tol:g}"

    def _c(self) -> rbpg_strategy:
        kind = {"direct": 0, "df": 1, "rank": 2}[self.kind]
        return rbpg_strategy(kind, self.split_index, self.rank_tol)


@dataclass
class ElmParams:
    inputs: int = 1
    hidden_nodes: int = 1
    outputs: int = 1
    seed: int = 0


@dataclass
class HiddenLayer:
    weights: np.ndarray  # inputs x L
    biases: np.ndarray   # 1 x L


@dataclass
class ElmModel:
    params: ElmParams
    hidden: HiddenLayer
    beta: np.ndarray     # L x m, original node order


@dataclass
class SolveDiagnostics:
    strategy: str = ""
    rank: int = 0
    rank_known: bool = False
    split_lo: int = 0
    split_hi: int = 0
    ridge_applied: bool = False
    fallback_to_direct: bool = False
    used_svd_path: bool = False
    solve_seconds: float = 0.0
    hidden_seconds: float = 0.0
    training_accuracy: float = -1.0

    def _fill(self, d: rbpg_diagnostics) -> "SolveDiagnostics":
        self.rank = int(d.rank)
        self.rank_known = bool(d.rank_known)
        self.split_lo = int(d.split_lo)
        self.split_hi = int(d.split_hi)
        self.ridge_applied = bool(d.ridge_applied)
        self.fallback_to_direct = bool(d.fallback_to_direct)
        self.used_svd_path = bool(d.used_svd_path)
        self.solve_seconds = float(d.solve_seconds)
        self.hidden_seconds = float(d.hidden_seconds)
        self.training_accuracy = float(d.training_accuracy)
        return self


@dataclass
class ColumnPermutation:
    order: List[int] = field(default_factory=list)
    rank: int = 0
    tolerance: float = 0.0


@dataclass
class RankRevealingFactor:
    permutation: ColumnPermutation
    factor: np.ndarray


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


class Context:
    """One device context (stream + workspace) of the native library."""

    def __init__(self, device: int = 0):
        self.lib = _native.load()
        h = ctypes.c_void_p()
        st = rbpg_status()
        self.lib.rbpg_context_create(device, ctypes.byref(h), ctypes.byref(st))
        _raise(st)
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            self.lib.rbpg_context_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        st = rbpg_status()
        self.lib.rbpg_context_set_stream(self.handle, ctypes.c_void_p(stream_ptr or None), ctypes.byref(st))
        _raise(st)

    def synchronize(self) -> None:
        st = rbpg_status()
        self.lib.rbpg_context_synchronize(self.handle, ctypes.byref(st))
        _raise(st)

    def set_profiling(self, enable: bool) -> None:
        """Per-kernel-class CUDA-event timing on the context stream (resets counters)."""
        st = rbpg_status()
        self.lib.rbpg_context_set_profiling(self.handle, int(enable), ctypes.byref(st))
        _raise(st)

    def profile(self, name: str):
        """(total_ms, launches) recorded for kernel class `name` since profiling was enabled."""
        ms = ctypes.c_double()
        cnt = ctypes.c_uint64()
        st = rbpg_status()
        self.lib.rbpg_context_profile_get(self.handle, name.encode(), ctypes.byref(ms), ctypes.byref(cnt),
                                          ctypes.byref(st))
        _raise(st)
        return float(ms.value), int(cnt.value)

    @property
    def launch_count(self) -> int:
        return int(self.lib.rbpg_context_launch_count(self.handle))


_ctx_lock = threading.Lock()
_contexts = {}


def _torch_stream(device) -> int:
    """Handle of torch's current stream on `device` for the device entry points.  torch's default
    stream is the legacy NULL stream (handle 0), which rbpg_context_set_stream would read as "the
    context's own (non-blocking) stream" -- unordered with torch's work -- so it is passed as
    cudaStreamLegacy (0x1) instead."""
    import torch

    return torch.cuda.current_stream(device).cuda_stream or 1


def context(device: int = 0) -> Context:
    with _ctx_lock:
        c = _contexts.get(device)
        if c is None:
            c = Context(device)
            _contexts[device] = c
        return c


def _f64(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    return np.ascontiguousarray(a)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check_matrix(a: np.ndarray) -> None:
    # DenseMatrix constructor contract (matrix.cpp:28-50)
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ShapeError(f"DenseMatrix dimensions must be positive, got {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("DenseMatrix data contains non-finite entries")


# ---------------------------------------------------------------------------
# reference API (host arrays)
# ---------------------------------------------------------------------------


def init_hidden(params: ElmParams) -> HiddenLayer:
    """elm.cpp:74-91 (bit-identical: std::mt19937_64 is standardised)."""
    lib = _native.load()
    if params.inputs < 1 or params.hidden_nodes < 1 or params.outputs < 1:
        raise ValueError("ElmParams: inputs, hidden_nodes and outputs must be >= 1")
    w = np.empty((params.inputs, params.hidden_nodes))
    b = np.empty((1, params.hidden_nodes))
    st = rbpg_status()
    lib.rbpg_init_hidden(params.inputs, params.hidden_nodes, params.outputs, params.seed, _ptr(w), _ptr(b),
                         ctypes.byref(st))
    _raise(st)
    return HiddenLayer(w, b)


def hidden_matrix(hidden: HiddenLayer, x, ctx: Optional[Context] = None) -> np.ndarray:
    """H = sigmoid(X W + b) on the device (K1; elm.cpp:93-106)."""
    ctx = ctx or context()
    x = _f64(x)
    w = _f64(hidden.weights)
    b = _f64(hidden.biases)
    d, l = w.shape
    h = np.empty((x.shape[0], l))
    st = rbpg_status()
    ctx.lib.rbpg_hidden_matrix(ctx.handle, _ptr(w), _ptr(b), d, l, _ptr(x), x.shape[0], x.shape[1], _ptr(h),
                               ctypes.byref(st))
    _raise(st)
    return h


def gram(a, ctx: Optional[Context] = None) -> np.ndarray:
    """a^T a, exactly symmetric (K2; matrix.cpp:152-161)."""
    ctx = ctx or context()
    a = _f64(a)
    g = np.empty((a.shape[1], a.shape[1]))
    st = rbpg_status()
    ctx.lib.rbpg_gram(ctx.handle, _ptr(a), a.shape[0], a.shape[1], _ptr(g), ctypes.byref(st))
    _raise(st)
    return g


def rank_revealing_factor(a, tol: float = 0.0, ctx: Optional[Context] = None) -> RankRevealingFactor:
    """Diagonal-pivoted Cholesky of a^T a (K2 + K3; linalg.cpp:157-248)."""
    ctx = ctx or context()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.size == 0:
        raise ShapeError("rank_revealing_permutation: empty matrix")
    a = np.ascontiguousarray(a)
    n = a.shape[1]
    order = np.empty(n, dtype=np.uint64)
    rank = ctypes.c_size_t()
    tolv = ctypes.c_double()
    f = np.empty((n, n))
    st = rbpg_status()
    ctx.lib.rbpg_rank_revealing_factor(ctx.handle, _ptr(a), a.shape[0], n, float(tol), _ptr(order),
                                       ctypes.byref(rank), ctypes.byref(tolv), _ptr(f), ctypes.byref(st))
    _raise(st)
    return RankRevealingFactor(ColumnPermutation([int(v) for v in order], int(rank.value), float(tolv.value)), f)


def rank_revealing_permutation(a, tol: float = 0.0, ctx: Optional[Context] = None) -> ColumnPermutation:
    return rank_revealing_factor(a, tol, ctx).permutation


def solve_factored_gram(f: RankRevealingFactor, rhs, ctx: Optional[Context] = None) -> np.ndarray:
    """linalg.cpp:254-270."""
    ctx = ctx or context()
    rhs = _f64(rhs)
    n = len(f.permutation.order)
    order = np.asarray(f.permutation.order, dtype=np.uint64)
    fac = _f64(f.factor)
    out = np.empty_like(rhs)
    st = rbpg_status()
    ctx.lib.rbpg_solve_factored_gram(ctx.handle, _ptr(fac), _ptr(order), n, f.permutation.rank, _ptr(rhs),
                                     rhs.shape[0], rhs.shape[1], _ptr(out), ctypes.byref(st))
    _raise(st)
    return out


def pinv_svd(a, tol: float = 0.0, ctx: Optional[Context] = None) -> np.ndarray:
    """SVD pseudo-inverse (linalg.cpp:68-87) on the device: block one-sided Jacobi SVD, singular
    values above rel * s_max inverted (rel = tol or max(rows, cols) * eps)."""
    ctx = ctx or context()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.size == 0:
        raise ShapeError("pinv_svd: empty matrix")
    a = np.ascontiguousarray(a)
    out = np.empty((a.shape[1], a.shape[0]))
    st = rbpg_status()
    ctx.lib.rbpg_pinv_svd(ctx.handle, _ptr(a), a.shape[0], a.shape[1], float(tol), _ptr(out), ctypes.byref(st))
    _raise(st)
    return out


def pseudo_inverse(h, tol: float = 0.0, ctx: Optional[Context] = None):
    """Rank-path pseudo-inverse H^+ = P (F F^T)^-1 P^T H^T (L x N) for full-rank H:
    the full-rank solve of elm.cpp:202-214 with right-hand side H^T.  Returns (hpinv, order, rank).
    Raises ValueError (invalid_argument, as solve_factored_gram at linalg.cpp:256-260) when rank < L."""
    ctx = ctx or context()
    h = np.asarray(h, dtype=np.float64)
    if h.ndim != 2 or h.size == 0:
        raise ShapeError("pseudo_inverse: empty matrix")
    h = np.ascontiguousarray(h)
    n, L = h.shape
    out = np.empty((L, n))
    order = np.empty(L, dtype=np.uint64)
    rank = ctypes.c_size_t()
    st = rbpg_status()
    ctx.lib.rbpg_pseudo_inverse(ctx.handle, _ptr(h), n, L, float(tol), _ptr(out), _ptr(order), ctypes.byref(rank),
                                ctypes.byref(st))
    _raise(st)
    return out, [int(v) for v in order], int(rank.value)


def solve_spd(m, rhs, ctx: Optional[Context] = None) -> np.ndarray:
    """linalg.cpp:99-155 (SpdFactor + solve)."""
    ctx = ctx or context()
    m = _f64(m)
    rhs = _f64(rhs)
    out = np.empty_like(rhs)
    st = rbpg_status()
    ctx.lib.rbpg_solve_spd(ctx.handle, _ptr(m), m.shape[0], m.shape[1], _ptr(rhs), rhs.shape[0], rhs.shape[1],
                           _ptr(out), ctypes.byref(st))
    _raise(st)
    return out


class SpdFactor:
    """linalg.hpp:45-60: Cholesky factor of a symmetric positive definite matrix, computed once on the
    device (SingularMatrix at construction, as the reference) and reused by every solve()."""

    def __init__(self, m, ctx: Optional[Context] = None):
        self.ctx = ctx or context()
        m = _f64(m)
        h = ctypes.c_void_p()
        st = rbpg_status()
        self.ctx.lib.rbpg_spd_create(self.ctx.handle, _ptr(m), m.shape[0], m.shape[1], ctypes.byref(h),
                                     ctypes.byref(st))
        _raise(st)
        self._h = h

    def dim(self) -> int:
        return int(self.ctx.lib.rbpg_spd_dim(self._h))

    def solve(self, rhs) -> np.ndarray:
        rhs = _f64(rhs)
        out = np.empty_like(rhs)
        st = rbpg_status()
        self.ctx.lib.rbpg_spd_solve(self._h, _ptr(rhs), rhs.shape[0], rhs.shape[1], _ptr(out), ctypes.byref(st))
        _raise(st)
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.ctx.lib.rbpg_spd_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def solve_block_split(h1, h2, y, ridge: float = 1e-8, diag: Optional[SolveDiagnostics] = None,
                      ctx: Optional[Context] = None) -> Tuple[np.ndarray, np.ndarray]:
    """elm.cpp:124-156: (beta1, beta2) of the block solve of [H1 H2] against Y (Gram of H2 + Schur
    complement, one ridge retry per block).  Raises ShapeError / SingularSplit like the reference."""
    ctx = ctx or context()
    h1, h2, y = _f64(h1), _f64(h2), _f64(y)
    b1 = np.empty((h1.shape[1], y.shape[1]))
    b2 = np.empty((h2.shape[1], y.shape[1]))
    d = rbpg_diagnostics()
    st = rbpg_status()
    ctx.lib.rbpg_solve_block_split(ctx.handle, _ptr(h1), h1.shape[0], h1.shape[1], _ptr(h2), h2.shape[0],
                                   h2.shape[1], _ptr(y), y.shape[0], y.shape[1], float(ridge), _ptr(b1), _ptr(b2),
                                   ctypes.byref(d), ctypes.byref(st))
    _raise(st)
    if diag is not None and d.ridge_applied:
        diag.ridge_applied = True
    return b1, b2


def _matmul(a, b, trans_a: bool, ctx: Optional[Context]) -> np.ndarray:
    ctx = ctx or context()
    a, b = _f64(a), _f64(b)
    out = np.empty((a.shape[1] if trans_a else a.shape[0], b.shape[1]))
    st = rbpg_status()
    ctx.lib.rbpg_matmul(ctx.handle, _ptr(a), a.shape[0], a.shape[1], int(trans_a), _ptr(b), b.shape[0], b.shape[1],
                        _ptr(out), ctypes.byref(st))
    _raise(st)
    return out


def matmul(a, b, ctx: Optional[Context] = None) -> np.ndarray:
    """matrix.cpp:69-77 on the DMMA GEMM."""
    return _matmul(a, b, False, ctx)


def matmul_at(a, b, ctx: Optional[Context] = None) -> np.ndarray:
    """matrix.cpp:79-87 (a^T b) on the DMMA GEMM."""
    return _matmul(a, b, True, ctx)


def solve_beta(h, y, strategy: SolverStrategy, diag: Optional[SolveDiagnostics] = None,
               ctx: Optional[Context] = None) -> np.ndarray:
    """elm.cpp:158-229 on a host H."""
    ctx = ctx or context()
    h = _f64(h)
    y = _f64(y)
    diag = diag if diag is not None else SolveDiagnostics()
    diag.strategy = strategy.describe()
    beta = np.empty((h.shape[1], y.shape[1]))
    s = strategy._c()
    d = rbpg_diagnostics()
    st = rbpg_status()
    ctx.lib.rbpg_solve_beta(ctx.handle, _ptr(h), h.shape[0], h.shape[1], _ptr(y), y.shape[0], y.shape[1],
                            ctypes.byref(s), _ptr(beta), ctypes.byref(d), ctypes.byref(st))
    _raise(st)
    acc = diag.training_accuracy
    diag._fill(d)
    diag.training_accuracy = acc
    diag.solve_seconds = diag.hidden_seconds = 0.0
    return beta


def solve_direct(h, y, diag: Optional[SolveDiagnostics] = None, ctx: Optional[Context] = None) -> np.ndarray:
    return solve_beta(h, y, SolverStrategy.direct(), diag if diag is not None else SolveDiagnostics(), ctx)


def train(params: ElmParams, x, y, strategy: SolverStrategy, ctx: Optional[Context] = None,
          return_order: bool = False):
    """elm.cpp:231-280.  Returns (ElmModel, SolveDiagnostics) [, order]."""
    ctx = ctx or context()
    x = _f64(x)
    y = _f64(y)
    L = max(params.hidden_nodes, 1)
    w = np.empty((max(params.inputs, 1), L))
    b = np.empty((1, L))
    beta = np.empty((L, max(params.outputs, 1)))
    order = np.zeros(L, dtype=np.uint64)
    s = strategy._c()
    d = rbpg_diagnostics()
    st = rbpg_status()
    ctx.lib.rbpg_train(ctx.handle, params.inputs, params.hidden_nodes, params.outputs, params.seed, _ptr(x),
                       x.shape[0], x.shape[1], _ptr(y), y.shape[0], y.shape[1], ctypes.byref(s), _ptr(w), _ptr(b),
                       _ptr(beta), _ptr(order) if return_order else None, ctypes.byref(d), ctypes.byref(st))
    _raise(st)
    diag = SolveDiagnostics(strategy=strategy.describe())._fill(d)
    model = ElmModel(params, HiddenLayer(w, b), beta)
    if return_order:
        return model, diag, [int(v) for v in order]
    return model, diag


def train_multi(params: ElmParams, x, y, strategy: SolverStrategy, devices=(0,), fixed_order: bool = False,
                return_order: bool = False):
    """Single-process multi-GPU train() (rbpg_train_multi): contiguous row shards over `devices`, one
    NCCL all-reduce of the packed augmented Gram (or all-gather + rank-order sum with fixed_order),
    replicated solve.  Returns (ElmModel, SolveDiagnostics) [, order]."""
    ctxs = [context(int(dv)) for dv in devices]
    arr = (ctypes.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
    lib = ctxs[0].lib
    x = _f64(x)
    y = _f64(y)
    L = max(params.hidden_nodes, 1)
    w = np.empty((max(params.inputs, 1), L))
    b = np.empty((1, L))
    beta = np.empty((L, max(params.outputs, 1)))
    order = np.zeros(L, dtype=np.uint64)
    s = strategy._c()
    d = rbpg_diagnostics()
    st = rbpg_status()
    lib.rbpg_train_multi(ctypes.cast(arr, ctypes.c_void_p), len(ctxs), params.inputs, params.hidden_nodes,
                         params.outputs, params.seed, _ptr(x), x.shape[0], x.shape[1], _ptr(y), y.shape[0],
                         y.shape[1], ctypes.byref(s), int(fixed_order), _ptr(w), _ptr(b), _ptr(beta), _ptr(order),
                         ctypes.byref(d), ctypes.byref(st))
    _raise(st)
    diag = SolveDiagnostics(strategy=strategy.describe())._fill(d)
    model = ElmModel(params, HiddenLayer(w, b), beta)
    if return_order:
        return model, diag, [int(v) for v in order]
    return model, diag


def predict(model: ElmModel, x, ctx: Optional[Context] = None) -> np.ndarray:
    """elm.cpp:282-284: sigmoid(X W + b) beta."""
    ctx = ctx or context()
    x = _f64(x)
    w = _f64(model.hidden.weights)
    b = _f64(model.hidden.biases)
    beta = _f64(model.beta)
    out = np.empty((x.shape[0], beta.shape[1]))
    st = rbpg_status()
    ctx.lib.rbpg_predict(ctx.handle, _ptr(w), _ptr(b), w.shape[0], w.shape[1], _ptr(beta), beta.shape[1], _ptr(x),
                         x.shape[0], x.shape[1], _ptr(out), ctypes.byref(st))
    _raise(st)
    return out


def accuracy(pred, y) -> float:
    """elm.cpp:286-300 (argmax, lowest index on ties)."""
    lib = _native.load()
    pred = _f64(pred)
    y = _f64(y)
    out = ctypes.c_double()
    st = rbpg_status()
    lib.rbpg_accuracy(_ptr(pred), pred.shape[0], pred.shape[1], _ptr(y), y.shape[0], y.shape[1], ctypes.byref(out),
                      ctypes.byref(st))
    _raise(st)
    return float(out.value)


def apply_permutation(a, p: ColumnPermutation) -> np.ndarray:
    """linalg.cpp:40-52 (pure data movement)."""
    a = np.asarray(a)
    if a.shape[1] != len(p.order):
        raise ShapeError(f"apply_permutation: matrix has {a.shape[1]} columns but permutation length is {len(p.order)}")
    return a[:, np.asarray(p.order, dtype=np.int64)].copy()


def invert_permutation_rows(b, p: ColumnPermutation) -> np.ndarray:
    """linalg.cpp:54-66."""
    b = np.asarray(b)
    if b.shape[0] != len(p.order):
        raise ShapeError(f"invert_permutation_rows: matrix has {b.shape[0]} rows but permutation length is {len(p.order)}")
    out = np.empty_like(b)
    out[np.asarray(p.order, dtype=np.int64)] = b
    return out


# ---------------------------------------------------------------------------
# synthetic inputs; host-side generators in the native library
# ---------------------------------------------------------------------------


def synth_classification(n: int, d: int, m: int, seed: int, teacher_seed: int, noise_sigma: float = 0.1,
                         row0: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    lib = _native.load()
    x = np.empty((n, d))
    t = np.empty((n, m))
    st = rbpg_status()
    lib.rbpg_synth_classification(row0, n, d, m, seed, teacher_seed, noise_sigma, _ptr(x), _ptr(t), ctypes.byref(st))
    _raise(st)
    return x, t


def synth_rank_deficient(n: int, base: int, m: int, seed: int, mix_seed: int, teacher_seed: int,
                         noise_sigma: float = 0.1) -> Tuple[np.ndarray, np.ndarray]:
    lib = _native.load()
    x = np.empty((n, 2 * base))
    t = np.empty((n, m))
    st = rbpg_status()
    lib.rbpg_synth_rank_deficient(n, base, m, seed, mix_seed, teacher_seed, noise_sigma, _ptr(x), _ptr(t),
                                  ctypes.byref(st))
    _raise(st)
    return x, t


def duplicate_nodes(hidden: HiddenLayer, ndup: int, seed: int) -> Tuple[HiddenLayer, np.ndarray, np.ndarray]:
    lib = _native.load()
    w = np.ascontiguousarray(hidden.weights, dtype=np.float64).copy()
    b = np.ascontiguousarray(hidden.biases, dtype=np.float64).copy()
    tgt = np.empty(ndup, dtype=np.uint64)
    src = np.empty(ndup, dtype=np.uint64)
    st = rbpg_status()
    lib.rbpg_duplicate_nodes(_ptr(w), _ptr(b), w.shape[0], w.shape[1], ndup, seed, _ptr(tgt), _ptr(src),
                             ctypes.byref(st))
    _raise(st)
    return HiddenLayer(w, b), tgt.astype(np.int64), src.astype(np.int64)


# ---------------------------------------------------------------------------
# device-resident entry points (torch CUDA tensors; used by bench.py and sharding)
# ---------------------------------------------------------------------------


def _tptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _ld(t) -> int:
    assert t.dim() == 2 and t.stride(1) == 1, "row-major 2-D tensor expected"
    return int(t.stride(0))


def train_device(x, t, params: ElmParams, strategy: SolverStrategy, hidden: Optional[HiddenLayer] = None,
                 ctx: Optional[Context] = None, return_order: bool = False):
    """train() on device-resident X (N x d) and T (N x m) torch float64 CUDA tensors.

    Returns (beta as a torch CUDA tensor, SolveDiagnostics, HiddenLayer) [, order].
    """
    import torch

    ctx = ctx or context(x.device.index or 0)
    ctx.set_stream(_torch_stream(x.device))
    hidden = hidden or init_hidden(params)
    w = _f64(hidden.weights)
    b = _f64(hidden.biases)
    L, m = w.shape[1], t.shape[1]
    beta = torch.empty((L, m), dtype=torch.float64, device=x.device)
    order = np.zeros(L, dtype=np.uint64)
    s = strategy._c()
    d = rbpg_diagnostics()
    st = rbpg_status()
    ctx.lib.rbpg_train_device(ctx.handle, _tptr(x), _ld(x), _tptr(t), _ld(t), x.shape[0], x.shape[1], L, m, _ptr(w),
                              _ptr(b), ctypes.byref(s), _tptr(beta), m, _ptr(order) if return_order else None,
                              ctypes.byref(d), ctypes.byref(st))
    _raise(st)
    diag = SolveDiagnostics(strategy=strategy.describe())._fill(d)
    if return_order:
        return beta, diag, hidden, [int(v) for v in order]
    return beta, diag, hidden


def gram_stage_device(x, t, w, b, g, htt, accumulate: bool = False, keep_h: bool = True,
                      ctx: Optional[Context] = None) -> None:
    """Stage 1 of the row-sharded path: local G (L x L) and H^T T (L x m) into torch tensors g, htt."""
    import torch

    ctx = ctx or context(x.device.index or 0)
    ctx.set_stream(_torch_stream(x.device))
    st = rbpg_status()
    ctx.lib.rbpg_gram_stage_device(ctx.handle, _tptr(x), _ld(x), _tptr(t), _ld(t), x.shape[0], x.shape[1],
                                   w.shape[1], t.shape[1], _tptr(w), _ld(w), _tptr(b), _tptr(g), _ld(g), _tptr(htt),
                                   _ld(htt), int(accumulate), int(keep_h), ctypes.byref(st))
    _raise(st)


def solve_stage_device(g, htt, n_total: int, strategy: SolverStrategy, ctx: Optional[Context] = None,
                       return_order: bool = False):
    """Stage 2 (replicated small solve on the all-reduced G, H^T T).  Returns (beta, diag[, order])."""
    import torch

    ctx = ctx or context(g.device.index or 0)
    ctx.set_stream(_torch_stream(g.device))
    L, m = htt.shape
    beta = torch.empty((L, m), dtype=torch.float64, device=g.device)
    order = np.zeros(L, dtype=np.uint64)
    s = strategy._c()
    d = rbpg_diagnostics()
    st = rbpg_status()
    ctx.lib.rbpg_solve_stage_device(ctx.handle, _tptr(g), _ld(g), _tptr(htt), _ld(htt), L, m, n_total,
                                    ctypes.byref(s), _tptr(beta), m, _ptr(order) if return_order else None,
                                    ctypes.byref(d), ctypes.byref(st))
    _raise(st)
    diag = SolveDiagnostics(strategy=strategy.describe())._fill(d)
    if return_order:
        return beta, diag, [int(v) for v in order]
    return beta, diag


def gram_stage_device_aug(x, t, w, b, gaug, accumulate: bool = False, keep_h: bool = True,
                          ctx: Optional[Context] = None) -> None:
    """Stage 1, augmented: gaug ((L+m) x (L+m) torch tensor) (+)= [H T]^T [H T] of the local rows."""
    import torch

    ctx = ctx or context(x.device.index or 0)
    ctx.set_stream(_torch_stream(x.device))
    st = rbpg_status()
    ctx.lib.rbpg_gram_stage_device_aug(ctx.handle, _tptr(x), _ld(x), _tptr(t), _ld(t), x.shape[0], x.shape[1],
                                       w.shape[1], t.shape[1], _tptr(w), _ld(w), _tptr(b), _tptr(gaug), _ld(gaug),
                                       int(accumulate), int(keep_h), ctypes.byref(st))
    _raise(st)


def solve_stage_device_aug(gaug, L: int, m: int, n_total: int, strategy: SolverStrategy,
                           ctx: Optional[Context] = None, return_order: bool = False):
    """Stage 2 on the all-reduced augmented Gram.  Returns (beta, diag[, order])."""
    import torch

    ctx = ctx or context(gaug.device.index or 0)
    ctx.set_stream(_torch_stream(gaug.device))
    beta = torch.empty((L, m), dtype=torch.float64, device=gaug.device)
    order = np.zeros(L, dtype=np.uint64)
    s = strategy._c()
    d = rbpg_diagnostics()
    st = rbpg_status()
    ctx.lib.rbpg_solve_stage_device_aug(ctx.handle, _tptr(gaug), _ld(gaug), L, m, n_total, ctypes.byref(s),
                                        _tptr(beta), m, _ptr(order) if return_order else None, ctypes.byref(d),
                                        ctypes.byref(st))
    _raise(st)
    diag = SolveDiagnostics(strategy=strategy.describe())._fill(d)
    if return_order:
        return beta, diag, [int(v) for v in order]
    return beta, diag


def accuracy_stage_device(x, t, w, b, beta, ctx: Optional[Context] = None) -> int:
    """Stage 3: number of local rows whose argmax(H beta) matches argmax(T)."""
    import torch

    ctx = ctx or context(x.device.index or 0)
    ctx.set_stream(_torch_stream(x.device))
    hits = ctypes.c_uint64()
    st = rbpg_status()
    ctx.lib.rbpg_accuracy_stage_device(ctx.handle, _tptr(x), _ld(x), _tptr(t), _ld(t), x.shape[0], x.shape[1],
                                       w.shape[1], t.shape[1], _tptr(w), _ld(w), _tptr(b), _tptr(beta), _ld(beta),
                                       ctypes.byref(hits), ctypes.byref(st))
    _raise(st)
    return int(hits.value)


def gram_device(a, g, accumulate: bool = False, ctx: Optional[Context] = None) -> None:
    """g (L x L torch tensor) (+)= a^T a for a device matrix a (rows x L)."""
    import torch

    ctx = ctx or context(a.device.index or 0)
    ctx.set_stream(_torch_stream(a.device))
    st = rbpg_status()
    ctx.lib.rbpg_gram_device(ctx.handle, _tptr(a), _ld(a), a.shape[0], a.shape[1], _tptr(g), _ld(g), int(accumulate),
                             ctypes.byref(st))
    _raise(st)


def gram_int8_device(a, g, accumulate: bool = False, ctx: Optional[Context] = None) -> None:
    """g (+)= a^T a with the train path's INT8 digit-plane Gram kernel (k_ozaki.cu) on any device matrix."""
    ctx = ctx or context(a.device.index or 0)
    ctx.set_stream(_torch_stream(a.device))
    st = rbpg_status()
    ctx.lib.rbpg_gram_int8_device(ctx.handle, _tptr(a), _ld(a), a.shape[0], a.shape[1], _tptr(g), _ld(g),
                                  int(accumulate), ctypes.byref(st))
    _raise(st)


def pseudo_inverse_stage_device(g, h, n_total: int, tol: float = 0.0, ctx: Optional[Context] = None):
    """Row-sharded H^+: from the all-reduced Gram g (L x L) of all n_total rows, this shard's column
    block H^+[:, local rows] (L x n_local torch tensor) for the local rows h (n_local x L).
    Returns (block, order, rank)."""
    import torch

    ctx = ctx or context(g.device.index or 0)
    ctx.set_stream(_torch_stream(g.device))
    L = g.shape[0]
    n_local = h.shape[0]
    out = torch.empty((L, max(n_local, 1) + (max(n_local, 1) & 1)), dtype=torch.float64, device=g.device)
    order = np.zeros(L, dtype=np.uint64)
    rank = ctypes.c_size_t()
    st = rbpg_status()
    ctx.lib.rbpg_pseudo_inverse_stage_device(ctx.handle, _tptr(g), _ld(g), n_total, _tptr(h), _ld(h), n_local, L,
                                             float(tol), _tptr(out), _ld(out), _ptr(order), ctypes.byref(rank),
                                             ctypes.byref(st))
    _raise(st)
    return out[:, :n_local], [int(v) for v in order], int(rank.value)


def predict_device(x, w, b, beta, scores=None, labels=None, ctx: Optional[Context] = None) -> None:
    """Batched predict (elm.cpp:282-284, arg-max rule elm.cpp:291-296) on device tensors: the fused
    sigma(X W + b) beta kernel writes scores (n x m float64) and/or labels (n int32); H is never stored."""
    ctx = ctx or context(x.device.index or 0)
    ctx.set_stream(_torch_stream(x.device))
    m = beta.shape[1]
    st = rbpg_status()
    ctx.lib.rbpg_predict_device(ctx.handle, _tptr(x), _ld(x), x.shape[0], x.shape[1], _tptr(w), _ld(w), _tptr(b),
                                w.shape[1], _tptr(beta), _ld(beta), m, _tptr(scores) if scores is not None else None,
                                _ld(scores) if scores is not None else 0,
                                _tptr(labels) if labels is not None else None, ctypes.byref(st))
    _raise(st)


def predict_labels_device(x, w, b, beta, labels, ctx: Optional[Context] = None) -> None:
    predict_device(x, w, b, beta, labels=labels, ctx=ctx)


def pack_lower_device(g, packed, ctx: Optional[Context] = None) -> None:
    """packed (n(n+1)/2 float64) <- lower triangle of the square device tensor g (row-major order)."""
    ctx = ctx or context(g.device.index or 0)
    ctx.set_stream(_torch_stream(g.device))
    st = rbpg_status()
    ctx.lib.rbpg_pack_lower_device(ctx.handle, _tptr(g), _ld(g), g.shape[0], _tptr(packed), ctypes.byref(st))
    _raise(st)


def unpack_lower_device(packed, g, ctx: Optional[Context] = None) -> None:
    """g (n x n, exactly symmetric) <- the packed lower triangle."""
    ctx = ctx or context(g.device.index or 0)
    ctx.set_stream(_torch_stream(g.device))
    st = rbpg_status()
    ctx.lib.rbpg_unpack_lower_device(ctx.handle, _tptr(packed), g.shape[0], _tptr(g), _ld(g), ctypes.byref(st))
    _raise(st)


def sum_parts_device(parts, out, ctx: Optional[Context] = None) -> None:
    """out = ((parts[0] + parts[1]) + parts[2]) + ... (parts: nparts x count, contiguous rows)."""
    ctx = ctx or context(parts.device.index or 0)
    ctx.set_stream(_torch_stream(parts.device))
    st = rbpg_status()
    ctx.lib.rbpg_sum_parts_device(ctx.handle, _tptr(parts), parts.stride(0), parts.shape[0], parts.shape[1],
                                  _tptr(out), ctypes.byref(st))
    _raise(st)
