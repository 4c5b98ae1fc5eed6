"""Pins the oracle restatement (oracle/rbpelm_oracle.cpp) against the REFERENCE'S OWN CODE.

oracle/_ref/librbpelm_ref.so is the reference's src/matrix.cpp, src/linalg.cpp and src/elm.cpp compiled
unedited where they lie under /root/reference, against a stand-in for the absent Eigen headers
(oracle/eigen_standin) -- so the pivot search, swaps, rank stop, tolerances, ridge retries, fallbacks and
error paths below are executed by the reference's code, and only the dense primitives (products, rank
updates, triangular solves, SVD) are the stand-in's.  Those primitives sum in increasing index order with
separately rounded multiplies and adds, which is also the oracle's order, so every Cholesky-based path
must agree BIT FOR BIT; the SVD fallback (two different Jacobi implementations of the same definition)
agrees to rounding.

The library is built here (where /root/reference exists) and travels to the GPU box inside oracle/_ref/;
without either the tests skip and tests/test_reference_golden.py's committed vectors stand in.
"""
import numpy as np
import pytest

import oracle
from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference library neither built nor buildable here")

DIAG_KEYS = ("rank", "rank_known", "split_lo", "split_hi", "ridge_applied", "fallback_to_direct", "used_svd_path")


def same_diag(a, b):
    return all(a[k] == b[k] for k in DIAG_KEYS)


def failure(mod, fn, *args, **kw):
    try:
        getattr(mod, fn)(*args, **kw)
    except oracle.OracleFailure as e:  # ref re-executes oracle.py's marshalling: its own class object
        return e.code, str(e).split(": ", 1)[1], e.pivot_index, e.block
    except ref.ReferenceFailure as e:
        return e.code, str(e).split(": ", 1)[1], e.pivot_index, e.block
    return None


@pytest.mark.parametrize("shape", [(2000, 16, 200, 2), (900, 8, 130, 3), (700, 5, 64, 4), (300, 3, 65, 2)],
                         ids=["C1", "3panels", "1panel", "panel+1"])
def test_train_rank_path_bitwise(shape):
    n, d, L, m = shape
    x, t = oracle.synth_classification(n, d, m, 1001, 2001)
    r = ref.train(d, L, m, 3001, x, t, "rank")
    o = oracle.train(d, L, m, 3001, x, t, "rank")
    assert np.array_equal(r["w"], o["w"]) and np.array_equal(r["b"], o["b"])  # init_hidden, elm.cpp:74-91
    assert r["order"] == o["order"] and r["diag"]["rank"] == o["diag"]["rank"] == L
    assert np.array_equal(r["beta"], o["beta"]), "beta differs from the reference's code"
    assert same_diag(r["diag"], o["diag"])
    assert r["diag"]["training_accuracy"] == o["diag"]["training_accuracy"]
    xt, _ = oracle.synth_classification(500, d, m, 1101, 2001)
    assert np.array_equal(ref.predict(r["w"], r["b"], r["beta"], xt), oracle.predict(o["w"], o["b"], o["beta"], xt))


def test_hidden_gram_factor_bitwise():
    x, _ = oracle.synth_classification(1200, 12, 2, 7, 8)
    w, b = oracle.init_hidden(12, 150, 2, 99)
    hr, ho = ref.hidden_matrix(w, b, x), oracle.hidden_matrix(w, b, x)
    assert np.array_equal(hr, ho)
    assert np.array_equal(ref.gram(hr), oracle.gram(ho))
    fr, fo = ref.rank_revealing_factor(hr), oracle.rank_revealing_factor(ho)
    assert fr[0] == fo[0] and fr[1] == fo[1] == 150 and fr[2] == fo[2]
    assert np.array_equal(fr[3], fo[3]), "factor F differs"
    rhs = np.random.default_rng(3).random((150, 4))
    assert np.array_equal(ref.solve_factored_gram(fr[3], fr[0], fr[1], rhs),
                          oracle.solve_factored_gram(fo[3], fo[0], fo[1], rhs))


def deficient_h(n=1500, d=24, L=300, dup=100, seed=5):
    """Hidden matrix with `dup` exact duplicate nodes (same W column and b): BASELINE C3's construction."""
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    x[:, d // 2:] = x[:, :d // 2] @ rng.random((d // 2, d - d // 2))  # dependent features
    w, b = oracle.init_hidden(d, L, 5, 77)
    w[:, L - dup:] = w[:, :dup]
    b[:, L - dup:] = b[:, :dup]
    y = np.eye(5)[rng.integers(0, 5, n)]
    return oracle.hidden_matrix(w, b, x), y


@pytest.mark.parametrize("kind,kw", [
    ("rank", dict(rank_tol=1e-6)),   # rank <= 200 of 300: Schur block path + ridge retry (elm.cpp:124-156, 29-49)
    ("rank", dict()),                # default tolerance: the stop among exact twins is decided by rounding
    ("df", dict(split_index=120)),
    ("df", dict(split_index=250)),
], ids=["rank-tol1e-6", "rank-default", "df120", "df250"])
def test_rank_deficient_paths_bitwise(kind, kw):
    h, y = deficient_h()
    br, dr, orr = ref.solve_beta(h, y, kind, **kw)
    bo, do, oo = oracle.solve_beta(h, y, kind, **kw)
    assert same_diag(dr, do), (dr, do)
    assert orr == oo, "pivot order (incl. the order among exact twins) differs"
    assert np.array_equal(br, bo)
    if kw.get("rank_tol"):
        assert 150 < dr["rank"] <= 200 and dr["ridge_applied"]  # 100 exact twins (+ near-dependent nodes)


def test_exact_ties_keep_lowest_index():
    """Equal diagonals: strict '>' (linalg.cpp:209) keeps the lowest index; the reference's code and the
    restatement must walk the same order through a Gram full of exact ties."""
    rng = np.random.default_rng(11)
    base = rng.random((400, 6))
    a = np.hstack([base, base[:, ::-1], base[:, :3]])  # every column has 1-2 exact twins
    fr, fo = ref.rank_revealing_factor(a, 1e-8), oracle.rank_revealing_factor(a, 1e-8)
    assert fr[0] == fo[0] and fr[1] == fo[1] == 6
    assert np.array_equal(fr[3], fo[3])
    z = np.zeros((5, 4))
    fr, fo = ref.rank_revealing_factor(z), oracle.rank_revealing_factor(z)
    assert fr[1] == fo[1] == 0 and fr[0] == fo[0] == [0, 1, 2, 3]  # all-zero: rank 0, identity (linalg.cpp:189-193)


def test_direct_and_svd_paths():
    rng = np.random.default_rng(2)
    h, y = rng.random((500, 80)), rng.random((500, 3))
    br, dr, _ = ref.solve_beta(h, y, "direct")
    bo, do, _ = oracle.solve_beta(h, y, "direct")
    assert same_diag(dr, do) and not dr["used_svd_path"]
    assert np.array_equal(br, bo)  # normal equations through SpdFactor
    h2, y2 = rng.random((40, 60)), rng.random((40, 3))  # N < L: the SVD pseudo-inverse path (elm.cpp:108-122)
    br, dr, _ = ref.solve_beta(h2, y2, "direct")
    bo, do, _ = oracle.solve_beta(h2, y2, "direct")
    assert same_diag(dr, do) and dr["used_svd_path"]
    assert np.linalg.norm(br - bo) <= 1e-12 * np.linalg.norm(bo)
    pr, po = ref.pinv_svd(h2), oracle.pinv_svd(h2)
    assert np.linalg.norm(pr - po) <= 1e-12 * np.linalg.norm(po)


def test_spd_and_block_split_bitwise():
    rng = np.random.default_rng(4)
    a = rng.random((90, 90))
    spd, rhs = a @ a.T + 90 * np.eye(90), rng.random((90, 5))
    assert np.array_equal(ref.solve_spd(spd, rhs), oracle.solve_spd(spd, rhs))  # two 64-wide panels
    assert np.array_equal(ref.matmul(a, rhs), oracle.matmul(a, rhs))
    h, y = rng.random((600, 70)), rng.random((600, 2))
    r1, r2, dr = ref.solve_block_split(h[:, :30], h[:, 30:], y)
    o1, o2, do = oracle.solve_block_split(h[:, :30], h[:, 30:], y)
    assert np.array_equal(r1, o1) and np.array_equal(r2, o2) and same_diag(dr, do)
    hd = np.hstack([h[:, :30], h[:, :30]])  # D block singular even after... the ridge rescues it
    r1, r2, dr = ref.solve_block_split(hd[:, :30], hd[:, 30:], y)
    o1, o2, do = oracle.solve_block_split(hd[:, :30], hd[:, 30:], y)
    assert np.array_equal(r1, o1) and np.array_equal(r2, o2) and same_diag(dr, do) and dr["ridge_applied"]


def test_error_behaviour_identical():
    rng = np.random.default_rng(6)
    a = rng.random((50, 50))
    spd, rhs = a @ a.T + 50 * np.eye(50), rng.random((50, 4))
    h, y = rng.random((100, 20)), rng.random((100, 2))
    x, t = oracle.synth_classification(50, 4, 2, 1, 2)
    cases = [
        ("solve_spd", (a[:, :40], rhs), {}),                       # ShapeError, not square
        ("solve_spd", (a, rhs), {}),                               # invalid_argument, not symmetric
        ("solve_spd", (spd, rhs[:10]), {}),                        # ShapeError, rhs rows
        ("solve_spd", (np.ones((4, 4)), np.ones((4, 1))), {}),     # SingularMatrix at index 1
        ("rank_revealing_factor", (h, -1.0), {}),                  # negative tolerance
        ("rank_revealing_factor", (h, float("nan")), {}),
        ("solve_factored_gram", (np.eye(4), [0, 1, 2, 3], 3, np.ones((4, 1))), {}),  # rank-deficient factor
        ("train", (4, 60, 2, 9, x, t, "rank"), {}),                # N < L on a block strategy
        ("train", (4, 20, 2, 9, x, t, "df", 0), {}),               # df split out of range
        ("train", (4, 20, 2, 9, x, t, "df", 20), {}),
        ("train", (5, 20, 2, 9, x, t, "rank"), {}),                # feature count mismatch
        ("train", (4, 20, 3, 9, x, t, "rank"), {}),                # output count mismatch
        ("train", (4, 20, 2, 9, x, t[:40], "rank"), {}),           # row mismatch
        ("matmul", (a, rhs[:10]), {}),
    ]
    for fn, args, kw in cases:
        fr, fo = failure(ref, fn, *args, **kw), failure(oracle, fn, *args, **kw)
        assert fr is not None, f"{fn}{args[2:]}: the reference did not raise"
        assert fr == fo, (fn, fr, fo)


def test_baseline_c2_bitwise():
    """BASELINE configs[1] (N=50000, d=64, L=1000, m=10; 16 panels) at full size: the restatement's
    blocked, threaded loops against the reference's own code -- pivot order, rank, beta and the
    training accuracy bit for bit (~70 s: the reference library is scalar and single-threaded)."""
    n, d, L, m = 50000, 64, 1000, 10
    x, t = oracle.synth_classification(n, d, m, 1001, 2001)
    o = oracle.train(d, L, m, 3001, x, t, "rank")
    r = ref.train(d, L, m, 3001, x, t, "rank")
    assert r["order"] == o["order"] and r["diag"]["rank"] == o["diag"]["rank"] == L
    assert np.array_equal(r["beta"], o["beta"])
    assert r["diag"]["training_accuracy"] == o["diag"]["training_accuracy"]


def test_reference_unit_suite_passes_on_the_standin_build():
    """The reference's own doctest suite (proj/tests/test_{matrix,linalg,elm,data,bench}.cpp, compiled
    unedited against oracle/doctest_standin) passes on the reference sources built with the Eigen
    stand-in: 50 test cases, every assertion -- the build that pins the oracle satisfies the
    reference's own known-answer and tolerance tests."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(ref.LIB), "unit_tests_ref")
    if not os.path.exists(exe):
        if not os.path.isdir(ref.REFERENCE_SRC):
            pytest.skip("unit_tests_ref not built and /root/reference absent")
        subprocess.run(["make", "-s", "-C", ref.HERE, "refunit"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout[-400:])
    assert out.returncode == 0, out.stdout[-2000:]
    assert "| 0 failed" in out.stdout and "test cases: " in out.stdout
    cases = int(out.stdout.split("test cases: ")[1].split(" ")[0])
    assert cases >= 42  # 50 with the bench tests (nlohmann json available), 42 without


def test_pseudo_inverse_definition_bitwise():
    """H+ = P (F F^T)^-1 P^T H^T is not computed by the reference's rank path; the oracle
    defines it as the full-rank solve (elm.cpp:202-214) with right-hand side H^T.  Composed here from the
    reference's own rank_revealing_factor / solve_factored_gram / row scatter, it must equal
    oracle.pseudo_inverse bit for bit, and satisfy the reference's pinv_svd to rounding."""
    x, _ = oracle.synth_classification(700, 10, 2, 21, 22)
    w, b = ref.init_hidden(10, 90, 2, 23)
    h = ref.hidden_matrix(w, b, x)
    order, rank, _, f, _ = ref.rank_revealing_factor(h)
    assert rank == 90
    xs = ref.solve_factored_gram(f, order, rank, np.ascontiguousarray(h.T[order]))
    hp = np.empty_like(xs)
    hp[order] = xs  # invert_permutation_rows, linalg.cpp:54-66
    hp_o, order_o, rank_o = oracle.pseudo_inverse(h)
    assert order_o == order and rank_o == rank
    assert np.array_equal(hp, hp_o)
    ps = ref.pinv_svd(h)
    assert np.linalg.norm(hp - ps) <= 1e-8 * np.linalg.norm(ps)
