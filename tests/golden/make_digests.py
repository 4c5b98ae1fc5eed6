"""Regenerate tests/golden/oracle_digests.json: SHA-256 digests of the oracle's outputs (Gram, pivot
order, factor, solve, beta, H^+) on seeded inputs.  The digests pin the oracle bitwise: a change to
its loop structure (blocking, threading, packing) must reproduce them exactly.

  python tests/golden/make_digests.py [path/to/liboracle_rbpelm.so]

The committed digests were produced by the round-1 oracle (scalar loops), so the current blocked /
threaded oracle is checked against that straightforward transcription."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

CASES = [  # (n, d, L, m, seed)
    (2000, 16, 200, 2, 11),
    (3000, 24, 333, 5, 12),
    (1500, 40, 700, 3, 13),
    (600, 8, 150, 4, 14),    # small d: rank-deficient at the default tolerance
]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes()).hexdigest()


def compute():
    out = {}
    for n, d, L, m, seed in CASES:
        rng = np.random.default_rng(seed)
        x = rng.uniform(0.0, 1.0, (n, d))
        t = np.eye(m)[rng.integers(0, m, n)]
        w, b = oracle.init_hidden(d, L, m, seed)
        h = oracle.hidden_matrix(w, b, x)
        g = oracle.gram(h)
        g4 = oracle.gram(h, 4)
        order, rank, tol, f, _ = oracle.factor_gram(g, n)
        r = oracle.train(d, L, m, seed, x, t, "rank")
        key = f"{n}x{d}x{L}x{m}"
        out[key] = {"h": digest(h), "gram": digest(g), "gram4": digest(g4), "order": order, "rank": rank,
                    "factor": digest(f), "beta": digest(r["beta"]), "train_order": r["order"],
                    "accuracy": r["diag"]["training_accuracy"]}
        if rank == L:
            rhs = (h.T @ t)[order]
            out[key]["solve"] = digest(oracle.solve_factored_gram(f, order, rank, rhs))
            out[key]["pinv"] = digest(oracle.pseudo_inverse(h)[0])
        out[key]["spd"] = digest(oracle.solve_spd(g + np.eye(L) * 1e-3 * np.trace(g) / L, h.T @ t))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1:
        oracle.LIB = sys.argv[1]
    oracle.set_threads(4)
    res = compute()
    json.dump(res, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_digests.json"), "w"),
              indent=0)
    print("wrote oracle_digests.json", {k: v["rank"] for k, v in res.items()})
