"""Regenerate tests/golden/reference_golden.json from the REFERENCE'S OWN CODE: oracle/_ref/librbpelm_ref.so,
i.e. /root/reference/proj/src/{matrix,linalg,elm}.cpp compiled unedited against oracle/eigen_standin
(`make -C oracle reflib`; needs /root/reference).  Inputs are the seeded generators of SURVEY 8(d)
(oracle.synth_classification: a pure function of its seeds), so only outputs are stored: pivot order,
rank, diagnostics, beta as IEEE-754 hex, arg-max labels of seeded test rows, and SHA-256 digests of the
big arrays (H, Gram, factor).  Run: python tests/golden/make_reference_golden.py"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (input generator only)
from oracle import ref  # noqa: E402

SEED_X, SEED_T, SEED_W, SEED_TEST = 1001, 2001, 3001, 1101
DIAG_KEYS = ("rank", "rank_known", "split_lo", "split_hi", "ridge_applied", "fallback_to_direct", "used_svd_path",
             "training_accuracy")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def hexes(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def train_case(name, n, d, L, m, tol=0.0, ntest=1000, kind="rank", split=0):
    x, t = oracle.synth_classification(n, d, m, SEED_X, SEED_T)
    r = ref.train(d, L, m, SEED_W, x, t, kind, split, tol)
    xt, _ = oracle.synth_classification(ntest, d, m, SEED_TEST, SEED_T)
    scores = ref.predict(r["w"], r["b"], r["beta"], xt)
    h = ref.hidden_matrix(r["w"], r["b"], x)
    f = ref.rank_revealing_factor(h, tol)
    return {"name": name, "kind": "train", "strategy": kind, "split": split, "n": n, "d": d, "L": L, "m": m, "tol": tol,
            "ntest": ntest,
            "order": r["order"], "diag": {k: r["diag"][k] for k in DIAG_KEYS},
            "beta_shape": list(r["beta"].shape), "beta_hex": hexes(r["beta"]),
            "train_labels": "".join(str(int(v)) for v in ref.predict(r["w"], r["b"], r["beta"], x).argmax(1)),
            "test_labels": "".join(str(int(v)) for v in scores.argmax(1)),
            "sha256": {"w": digest(r["w"]), "b": digest(r["b"]), "h": digest(h), "gram": digest(ref.gram(h)),
                       "factor": digest(f[3]), "test_scores": digest(scores)}}


def deficient_case(name, n, d, L, dup, m, tol):
    """Duplicate nodes (BASELINE C3's construction) through solve_beta on the H they produce."""
    x, t = oracle.synth_classification(n, d, m, SEED_X, SEED_T)
    w, b = ref.init_hidden(d, L, m, SEED_W)
    w[:, L - dup:] = w[:, :dup]
    b[:, L - dup:] = b[:, :dup]
    h = ref.hidden_matrix(w, b, x)
    beta, diag, order = ref.solve_beta(h, t, "rank", 0, tol)
    return {"name": name, "kind": "deficient", "n": n, "d": d, "L": L, "dup": dup, "m": m, "tol": tol,
            "order": order, "diag": {k: diag[k] for k in DIAG_KEYS if k != "training_accuracy"},
            "beta_shape": list(beta.shape), "beta_hex": hexes(beta),
            "fitted_sha256": digest(ref.matmul(h, beta)), "sha256": {"h": digest(h)}}


cases = [
    train_case("C1", 2000, 16, 200, 2),                 # BASELINE configs[0], 1000 seeded test rows
    # well-posed shapes (oracle pivot margin >= 1e-8, self-floor ~1e-11): a pivot order decided by
    # rounding noise could not be held to bit-exactness on any other arithmetic, real Eigen included
    train_case("three_panels", 900, 24, 130, 3, ntest=300),
    train_case("panel_plus_one", 600, 16, 65, 2, ntest=100),
    # the DF split and the direct strategy through the same train()
    train_case("df_split_40", 900, 24, 130, 3, ntest=300, kind="df", split=40),
    train_case("direct", 900, 24, 130, 3, ntest=300, kind="direct"),
    deficient_case("twins_tol1e-6", 1500, 12, 300, 100, 5, 1e-6),
]
out = {"generator": "tests/golden/make_reference_golden.py",
       "source": "reference proj/src/{matrix,linalg,elm}.cpp compiled unedited against oracle/eigen_standin "
                 "(sequential sums, -ffp-contract=off)",
       "seeds": {"x": SEED_X, "teacher": SEED_T, "w": SEED_W, "test": SEED_TEST}, "cases": cases}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")
json.dump(out, open(path, "w"), indent=0)
for c in cases:
    print(c["name"], c["diag"])
print("wrote", path, os.path.getsize(path), "bytes")
