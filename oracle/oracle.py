"""ctypes wrapper of liboracle_rbpelm.so (test infrastructure only)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char, c_double, c_int, c_size_t, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle_rbpelm.so")

KIND = {"direct": 0, "df": 1, "rank": 2}


class OracleError(ctypes.Structure):
    _fields_ = [("code", c_int), ("pivot_index", c_size_t), ("pivot_value", c_double), ("block", c_int),
                ("message", c_char * 256)]


class OracleDiag(ctypes.Structure):
    _fields_ = [("rank", c_size_t), ("rank_known", c_int), ("split_lo", c_size_t), ("split_hi", c_size_t),
                ("ridge_applied", c_int), ("fallback_to_direct", c_int), ("used_svd_path", c_int),
                ("solve_seconds", c_double), ("hidden_seconds", c_double), ("training_accuracy", c_double),
                ("min_pivot_margin", c_double)]


class OracleFailure(Exception):
    def __init__(self, err: OracleError):
        self.code = err.code
        self.pivot_index = err.pivot_index
        self.pivot_value = err.pivot_value
        self.block = err.block
        super().__init__(f"oracle error {err.code}: {err.message.decode(errors='replace')}")


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        _lib.oracle_set_threads.argtypes = [c_int]
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def _p(a):
    return a.ctypes.data_as(c_void_p)


def _f(a):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    return np.ascontiguousarray(a)


def _call(fn, *args):
    err = OracleError()
    rc = fn(*args, ctypes.byref(err))
    if rc != 0:
        raise OracleFailure(err)


def init_hidden(inputs, hidden, outputs, seed):
    w = np.empty((inputs, hidden))
    b = np.empty((1, hidden))
    _call(lib().oracle_init_hidden, c_size_t(inputs), c_size_t(hidden), c_size_t(outputs), c_uint64(seed), _p(w), _p(b))
    return w, b


def hidden_matrix(w, b, x):
    w, b, x = _f(w), _f(b), _f(x)
    h = np.empty((x.shape[0], w.shape[1]))
    _call(lib().oracle_hidden_matrix, _p(w), _p(b), c_size_t(w.shape[0]), c_size_t(w.shape[1]), _p(x),
          c_size_t(x.shape[0]), c_size_t(x.shape[1]), _p(h))
    return h


def gram(a, shards=1):
    a = _f(a)
    g = np.empty((a.shape[1], a.shape[1]))
    _call(lib().oracle_gram, _p(a), c_size_t(a.shape[0]), c_size_t(a.shape[1]), c_size_t(shards), _p(g))
    return g


def matmul(a, b):
    a, b = _f(a), _f(b)
    o = np.empty((a.shape[0], b.shape[1]))
    _call(lib().oracle_matmul, _p(a), c_size_t(a.shape[0]), c_size_t(a.shape[1]), _p(b), c_size_t(b.shape[0]),
          c_size_t(b.shape[1]), _p(o))
    return o


def pinv_svd(a, tol=0.0):
    a = _f(a)
    o = np.empty((a.shape[1], a.shape[0]))
    _call(lib().oracle_pinv_svd, _p(a), c_size_t(a.shape[0]), c_size_t(a.shape[1]), c_double(tol), _p(o))
    return o


def solve_spd(m, rhs):
    m, rhs = _f(m), _f(rhs)
    o = np.empty_like(rhs)
    _call(lib().oracle_solve_spd, _p(m), c_size_t(m.shape[0]), c_size_t(m.shape[1]), _p(rhs), c_size_t(rhs.shape[0]),
          c_size_t(rhs.shape[1]), _p(o))
    return o


def rank_revealing_factor(a, tol=0.0):
    """Returns (order, rank, tolerance, factor, min_margin)."""
    a = _f(a)
    n = a.shape[1]
    order = np.empty(n, dtype=np.uint64)
    rank = c_size_t()
    tv = c_double()
    mm = c_double()
    f = np.empty((n, n))
    _call(lib().oracle_rank_revealing_factor, _p(a), c_size_t(a.shape[0]), c_size_t(n), c_double(tol), _p(order),
          ctypes.byref(rank), ctypes.byref(tv), _p(f), ctypes.byref(mm))
    return [int(v) for v in order], int(rank.value), float(tv.value), f, float(mm.value)


def factor_gram(g, rows, tol=0.0):
    """Same factorisation on a precomputed Gram.  Returns (order, rank, tolerance, factor, min_margin)."""
    g = _f(g)
    n = g.shape[0]
    order = np.empty(n, dtype=np.uint64)
    rank = c_size_t()
    tv = c_double()
    mm = c_double()
    f = np.empty((n, n))
    _call(lib().oracle_factor_gram, _p(g), c_size_t(n), c_size_t(rows), c_double(tol), _p(order), ctypes.byref(rank),
          ctypes.byref(tv), _p(f), ctypes.byref(mm))
    return [int(v) for v in order], int(rank.value), float(tv.value), f, float(mm.value)


def solve_factored_gram(factor, order, rank, rhs):
    factor, rhs = _f(factor), _f(rhs)
    n = factor.shape[0]
    o = np.asarray(order, dtype=np.uint64)
    out = np.empty_like(rhs)
    _call(lib().oracle_solve_factored_gram, _p(factor), _p(o), c_size_t(n), c_size_t(rank), _p(rhs),
          c_size_t(rhs.shape[0]), c_size_t(rhs.shape[1]), _p(out))
    return out


def pseudo_inverse(h, tol=0.0):
    """Rank-path H^+ = P (F F^T)^-1 P^T H^T (full rank only).  Returns (hpinv, order, rank);
    raises OracleFailure (code 2, invalid_argument) when rank < cols."""
    h = _f(h)
    n, l = h.shape
    out = np.empty((l, n))
    order = np.empty(l, dtype=np.uint64)
    rank = c_size_t()
    _call(lib().oracle_pseudo_inverse, _p(h), c_size_t(n), c_size_t(l), c_double(tol), _p(out), _p(order),
          ctypes.byref(rank))
    return out, [int(v) for v in order], int(rank.value)


def solve_block_split(h1, h2, y, ridge=1e-8):
    h1, h2, y = _f(h1), _f(h2), _f(y)
    b1 = np.empty((h1.shape[1], y.shape[1]))
    b2 = np.empty((h2.shape[1], y.shape[1]))
    d = OracleDiag()
    _call(lib().oracle_solve_block_split, _p(h1), c_size_t(h1.shape[0]), c_size_t(h1.shape[1]), _p(h2),
          c_size_t(h2.shape[1]), _p(y), c_size_t(y.shape[1]), c_double(ridge), _p(b1), _p(b2), ctypes.byref(d))
    return b1, b2, _diag(d)


def _diag(d):
    return {k: getattr(d, k) for k, _ in OracleDiag._fields_}


def solve_beta(h, y, kind="rank", split_index=0, rank_tol=0.0, gram_shards=1):
    """Returns (beta, diag dict, order or None)."""
    h, y = _f(h), _f(y)
    beta = np.empty((h.shape[1], y.shape[1]))
    order = np.empty(h.shape[1], dtype=np.uint64)
    d = OracleDiag()
    _call(lib().oracle_solve_beta, _p(h), c_size_t(h.shape[0]), c_size_t(h.shape[1]), _p(y), c_size_t(y.shape[0]),
          c_size_t(y.shape[1]), c_int(KIND[kind]), c_size_t(split_index), c_double(rank_tol), c_size_t(gram_shards),
          _p(beta), _p(order), ctypes.byref(d))
    dd = _diag(d)
    return beta, dd, ([int(v) for v in order] if kind == "rank" and dd["rank_known"] else None)


def train(inputs, hidden, outputs, seed, x, y, kind="rank", split_index=0, rank_tol=0.0, gram_shards=1):
    """Returns dict(w, b, beta, order, diag)."""
    x, y = _f(x), _f(y)
    w = np.empty((inputs, hidden))
    b = np.empty((1, hidden))
    beta = np.empty((hidden, outputs))
    order = np.zeros(hidden, dtype=np.uint64)
    d = OracleDiag()
    _call(lib().oracle_train, c_size_t(inputs), c_size_t(hidden), c_size_t(outputs), c_uint64(seed), _p(x),
          c_size_t(x.shape[0]), c_size_t(x.shape[1]), _p(y), c_size_t(y.shape[0]), c_size_t(y.shape[1]),
          c_int(KIND[kind]), c_size_t(split_index), c_double(rank_tol), c_size_t(gram_shards), _p(w), _p(b), _p(beta),
          _p(order), ctypes.byref(d))
    return {"w": w, "b": b, "beta": beta, "order": [int(v) for v in order], "diag": _diag(d)}


def predict(w, b, beta, x):
    w, b, beta, x = _f(w), _f(b), _f(beta), _f(x)
    out = np.empty((x.shape[0], beta.shape[1]))
    _call(lib().oracle_predict, _p(w), _p(b), c_size_t(w.shape[0]), c_size_t(w.shape[1]), _p(beta),
          c_size_t(beta.shape[1]), _p(x), c_size_t(x.shape[0]), c_size_t(x.shape[1]), _p(out))
    return out


def accuracy(pred, y):
    pred, y = _f(pred), _f(y)
    out = c_double()
    _call(lib().oracle_accuracy, _p(pred), c_size_t(pred.shape[0]), c_size_t(pred.shape[1]), _p(y),
          c_size_t(y.shape[0]), c_size_t(y.shape[1]), ctypes.byref(out))
    return float(out.value)


def synth_classification(n, d, m, seed, teacher_seed, noise_sigma=0.1, row0=0):
    """SURVEY §8(d) synthetic classification rows [row0, row0 + n): the generator definition the
    product's rbpg_synth_classification implements, restated so that bench.py's CPU legs never load
    the product library.  Returns (X n x d, one-hot T n x m)."""
    x = np.empty((n, d))
    t = np.empty((n, m))
    _call(lib().oracle_synth_classification, c_size_t(row0), c_size_t(n), c_size_t(d), c_size_t(m), c_uint64(seed),
          c_uint64(teacher_seed), c_double(noise_sigma), _p(x), _p(t))
    return x, t


PHASES = ("hidden", "gram", "factor", "solve", "accuracy")


def train_phase_times(inputs, hidden, outputs, seed, x, y, ridge=1e-2):
    """Seconds per phase of train(rank) on the sample rows x, y (see oracle_train_phase_times):
    dict over PHASES plus 'rank'.  hidden/gram/accuracy are linear in the row count."""
    x, y = _f(x), _f(y)
    times = np.zeros(5)
    rank = c_size_t()
    _call(lib().oracle_train_phase_times, c_size_t(inputs), c_size_t(hidden), c_size_t(outputs), c_uint64(seed),
          _p(x), c_size_t(x.shape[0]), _p(y), c_double(ridge), _p(times), ctypes.byref(rank))
    out = dict(zip(PHASES, (float(v) for v in times)))
    out["rank"] = int(rank.value)
    return out
