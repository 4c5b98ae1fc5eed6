"""Golden vectors produced by the REFERENCE'S OWN CODE (tests/golden/reference_golden.json, written by
tests/golden/make_reference_golden.py from oracle/_ref/librbpelm_ref.so: the reference's matrix.cpp,
linalg.cpp and elm.cpp compiled unedited against the Eigen stand-in).  They travel with the repo, so
they pin both sides wherever /root/reference is absent:

  * CPU: the oracle restatement reproduces every vector bit for bit (beta, pivot order, rank,
    diagnostics, labels, SHA-256 of W, b, H, the Gram and the factor);
  * GPU (-m gpu): the B200 path through the C ABI gives the same pivot order, rank, diagnostics and
    labels, and beta within the north-star 1e-9 relative Frobenius error of the reference's beta.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.json")))
SEEDS = GOLD["seeds"]
TRAIN = [c for c in GOLD["cases"] if c["kind"] == "train"]
DEFICIENT = [c for c in GOLD["cases"] if c["kind"] == "deficient"]
FLAGS = ("rank", "rank_known", "split_lo", "split_hi", "ridge_applied", "fallback_to_direct", "used_svd_path")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def beta_of(c):
    return np.array([float.fromhex(v) for v in c["beta_hex"]]).reshape(c["beta_shape"])


def labels(scores):
    return "".join(str(int(v)) for v in np.asarray(scores).argmax(1))


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("c", TRAIN, ids=[c["name"] for c in TRAIN])
def test_oracle_reproduces_reference_train_vectors(c):
    x, t = oracle.synth_classification(c["n"], c["d"], c["m"], SEEDS["x"], SEEDS["teacher"])
    o = oracle.train(c["d"], c["L"], c["m"], SEEDS["w"], x, t, c["strategy"], c["split"], c["tol"])
    if c["strategy"] == "rank":
        assert o["order"] == c["order"]
    assert all(o["diag"][k] == c["diag"][k] for k in FLAGS)
    assert o["diag"]["training_accuracy"] == c["diag"]["training_accuracy"]
    assert np.array_equal(o["beta"], beta_of(c)), "oracle beta is not bitwise the reference's"
    h = oracle.hidden_matrix(o["w"], o["b"], x)
    f = oracle.rank_revealing_factor(h, c["tol"])
    got = {"w": digest(o["w"]), "b": digest(o["b"]), "h": digest(h), "gram": digest(oracle.gram(h)),
           "factor": digest(f[3])}
    xt, _ = oracle.synth_classification(c["ntest"], c["d"], c["m"], SEEDS["test"], SEEDS["teacher"])
    scores = oracle.predict(o["w"], o["b"], o["beta"], xt)
    got["test_scores"] = digest(scores)
    assert got == c["sha256"]
    assert labels(scores) == c["test_labels"]
    assert labels(oracle.predict(o["w"], o["b"], o["beta"], x)) == c["train_labels"]


@pytest.mark.parametrize("c", DEFICIENT, ids=[c["name"] for c in DEFICIENT])
def test_oracle_reproduces_reference_deficient_vectors(c):
    x, t = oracle.synth_classification(c["n"], c["d"], c["m"], SEEDS["x"], SEEDS["teacher"])
    w, b = oracle.init_hidden(c["d"], c["L"], c["m"], SEEDS["w"])
    w[:, c["L"] - c["dup"]:] = w[:, :c["dup"]]
    b[:, c["L"] - c["dup"]:] = b[:, :c["dup"]]
    h = oracle.hidden_matrix(w, b, x)
    assert digest(h) == c["sha256"]["h"]
    beta, diag, order = oracle.solve_beta(h, t, "rank", 0, c["tol"])
    assert order == c["order"] and all(diag[k] == c["diag"][k] for k in FLAGS)
    assert np.array_equal(beta, beta_of(c))
    assert digest(oracle.matmul(h, beta)) == c["fitted_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("c", TRAIN, ids=[c["name"] for c in TRAIN])
def test_b200_train_matches_reference_vectors(c):
    import paper_2011_02436_b200 as rb

    x, t = rb.synth_classification(c["n"], c["d"], c["m"], SEEDS["x"], SEEDS["teacher"])
    params = rb.ElmParams(c["d"], c["L"], c["m"], SEEDS["w"])
    strategy = {"rank": rb.SolverStrategy.rank_based(c["tol"]), "df": rb.SolverStrategy.df_split(c["split"]),
                "direct": rb.SolverStrategy.direct()}[c["strategy"]]
    model, diag, order = rb.train(params, x, t, strategy, return_order=True)
    assert digest(model.hidden.weights) == c["sha256"]["w"] and digest(model.hidden.biases) == c["sha256"]["b"]
    if c["strategy"] == "rank":
        assert order == c["order"], "pivot order differs from the reference's"
    assert diag.rank == c["diag"]["rank"] and diag.split_lo == c["diag"]["split_lo"]
    assert diag.rank_known == bool(c["diag"]["rank_known"]) and diag.used_svd_path == bool(c["diag"]["used_svd_path"])
    assert diag.split_hi == c["diag"]["split_hi"] and not diag.ridge_applied and not diag.fallback_to_direct
    assert diag.training_accuracy == c["diag"]["training_accuracy"]
    err = rel_fro(model.beta, beta_of(c))
    print(f"{c['name']}: beta rel vs the reference's {err:.3e}")
    assert err <= 1e-9  # north star: beta within relative Frobenius 1e-9
    xt, _ = rb.synth_classification(c["ntest"], c["d"], c["m"], SEEDS["test"], SEEDS["teacher"])
    assert labels(rb.predict(model, xt)) == c["test_labels"]
    assert labels(rb.predict(model, x)) == c["train_labels"]


@pytest.mark.gpu
@pytest.mark.parametrize("c", DEFICIENT, ids=[c["name"] for c in DEFICIENT])
def test_b200_rank_deficient_matches_reference_vectors(c):
    import paper_2011_02436_b200 as rb

    L, dup = c["L"], c["dup"]
    x, t = rb.synth_classification(c["n"], c["d"], c["m"], SEEDS["x"], SEEDS["teacher"])
    hid = rb.init_hidden(rb.ElmParams(c["d"], L, c["m"], SEEDS["w"]))
    hid.weights[:, L - dup:] = hid.weights[:, :dup]
    hid.biases[:, L - dup:] = hid.biases[:, :dup]
    h = rb.hidden_matrix(hid, x)
    assert np.array_equal(h[:, L - dup:], h[:, :dup])  # exact twins on the device too
    diag = rb.SolveDiagnostics()
    beta = rb.solve_beta(h, t, rb.SolverStrategy.rank_based(c["tol"]), diag)
    r = c["diag"]["rank"]
    assert diag.rank == r and diag.ridge_applied == bool(c["diag"]["ridge_applied"])
    assert diag.split_lo == c["diag"]["split_lo"] and diag.split_hi == c["diag"]["split_hi"]
    assert not diag.fallback_to_direct
    f = rb.rank_revealing_factor(h, c["tol"])
    cls = lambda j: j - (L - dup) if j >= L - dup else j  # noqa: E731  twin class of a node
    assert f.permutation.rank == r
    assert [cls(j) for j in f.permutation.order[:r]] == [cls(j) for j in c["order"][:r]]
    print("raw pivot order identical to the reference's:", list(f.permutation.order[:r]) == c["order"][:r])
    fit, fit_ref = h @ beta, h @ beta_of(c)  # beta itself is not unique at rank < L
    err = rel_fro(fit, fit_ref)
    print(f"{c['name']}: fitted values rel vs the reference's {err:.3e}")
    assert err < 1e-8 and (fit.argmax(1) == fit_ref.argmax(1)).all()
