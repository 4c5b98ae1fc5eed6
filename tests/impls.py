"""Two implementations behind one test-facing interface: the CPU oracle
(test infrastructure) and the B200 product (C ABI -> sm_100a kernels).

The reference's own unit/acceptance tests (proj/tests/*.cpp) are written once
against this interface and run on both: on the oracle in the CPU suite (pins
the restatement) and on the GPU in the `-m gpu` suite."""
from __future__ import annotations

import numpy as np

import oracle
import paper_2011_02436_b200 as rb

ShapeError = rb.ShapeError
SingularMatrix = rb.SingularMatrix
SingularSplit = rb.SingularSplit


def _translate(exc: oracle.OracleFailure):
    msg = str(exc)
    if exc.code == 1:
        return ShapeError(msg)
    if exc.code == 2:
        return ValueError(msg)
    if exc.code == 3:
        return SingularMatrix(exc.pivot_index, exc.pivot_value, msg)
    if exc.code == 4:
        return SingularSplit(exc.block, msg)
    return RuntimeError(msg)


class OracleImpl:
    name = "oracle"

    def _call(self, fn, *a, **k):
        try:
            return fn(*a, **k)
        except oracle.OracleFailure as e:
            raise _translate(e) from None

    def init_hidden(self, d, L, m, seed):
        return self._call(oracle.init_hidden, d, L, m, seed)

    def hidden_matrix(self, w, b, x):
        return self._call(oracle.hidden_matrix, w, b, x)

    def gram(self, a):
        return self._call(oracle.gram, a)

    def rrf(self, a, tol=0.0):
        order, rank, tolv, f, _ = self._call(oracle.rank_revealing_factor, a, tol)
        return order, rank, tolv, f

    def solve_spd(self, m, rhs):
        return self._call(oracle.solve_spd, m, rhs)

    def solve_factored_gram(self, factor, order, rank, rhs):
        return self._call(oracle.solve_factored_gram, factor, order, rank, rhs)

    def pinv_svd(self, a, tol=0.0):
        return self._call(oracle.pinv_svd, a, tol)

    def solve_beta(self, h, y, kind="rank", split=0, tol=0.0):
        beta, diag, _ = self._call(oracle.solve_beta, h, y, kind, split, tol)
        return beta, diag

    def train(self, d, L, m, seed, x, y, kind="rank", split=0, tol=0.0):
        r = self._call(oracle.train, d, L, m, seed, x, y, kind, split, tol)
        return r["beta"], r["diag"], r["w"], r["b"]

    def predict(self, w, b, beta, x):
        return self._call(oracle.predict, w, b, beta, x)

    def accuracy(self, pred, y):
        return self._call(oracle.accuracy, pred, y)


class B200Impl:
    name = "b200"

    def init_hidden(self, d, L, m, seed):
        h = rb.init_hidden(rb.ElmParams(d, L, m, seed))
        return h.weights, h.biases

    def hidden_matrix(self, w, b, x):
        return rb.hidden_matrix(rb.HiddenLayer(np.asarray(w, dtype=float), np.asarray(b, dtype=float).reshape(1, -1)), x)

    def gram(self, a):
        return rb.gram(a)

    def rrf(self, a, tol=0.0):
        f = rb.rank_revealing_factor(a, tol)
        return f.permutation.order, f.permutation.rank, f.permutation.tolerance, f.factor

    def solve_spd(self, m, rhs):
        return rb.solve_spd(m, rhs)

    def solve_factored_gram(self, factor, order, rank, rhs):
        perm = rb.ColumnPermutation(list(order), rank, 0.0)
        return rb.solve_factored_gram(rb.RankRevealingFactor(perm, np.asarray(factor, dtype=float)), rhs)

    def pinv_svd(self, a, tol=0.0):
        return rb.pinv_svd(a, tol)

    def _strategy(self, kind, split, tol):
        return {"rank": rb.SolverStrategy.rank_based(tol), "df": rb.SolverStrategy.df_split(split),
                "direct": rb.SolverStrategy.direct()}[kind]

    def _diag(self, d):
        return {"rank": d.rank, "rank_known": int(d.rank_known), "split_lo": d.split_lo, "split_hi": d.split_hi,
                "ridge_applied": int(d.ridge_applied), "fallback_to_direct": int(d.fallback_to_direct),
                "used_svd_path": int(d.used_svd_path), "training_accuracy": d.training_accuracy}

    def solve_beta(self, h, y, kind="rank", split=0, tol=0.0):
        diag = rb.SolveDiagnostics()
        beta = rb.solve_beta(h, y, self._strategy(kind, split, tol), diag)
        return beta, self._diag(diag)

    def train(self, d, L, m, seed, x, y, kind="rank", split=0, tol=0.0):
        model, diag = rb.train(rb.ElmParams(d, L, m, seed), x, y, self._strategy(kind, split, tol))
        return model.beta, self._diag(diag), model.hidden.weights, model.hidden.biases

    def predict(self, w, b, beta, x):
        model = rb.ElmModel(rb.ElmParams(), rb.HiddenLayer(np.asarray(w, dtype=float), np.asarray(b, dtype=float).reshape(1, -1)),
                            np.asarray(beta, dtype=float))
        return rb.predict(model, x)

    def accuracy(self, pred, y):
        return rb.accuracy(pred, y)


def rel_err(got, want):
    """reference tests' rel_err: max|got - want| / (1 + max|want|)"""
    got, want = np.asarray(got), np.asarray(want)
    return float(np.abs(got - want).max() / (1.0 + np.abs(want).max()))


def rel_fro(got, want):
    got, want = np.asarray(got), np.asarray(want)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def pinv(a, tol=0.0):
    """Independent SVD pseudoinverse (numpy LAPACK) with the reference's cut rule (linalg.cpp:68-87)."""
    a = np.asarray(a, dtype=float)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    rel = tol if tol > 0 else max(a.shape) * np.finfo(float).eps
    cut = rel * (s[0] if s.size else 0.0)
    inv = np.where((s > cut) & (s > 0), 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (vt.T * inv) @ u.T
