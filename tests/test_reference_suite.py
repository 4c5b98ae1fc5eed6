"""The reference's own unit and acceptance tests, ported (proj/tests/test_linalg.cpp,
test_elm.cpp, test_matrix.cpp, acceptance.cpp, src/checks.cpp).

Each test runs on the CPU oracle (CPU suite: pins the restatement against the
reference's known answers and tolerances) and on the B200 product (`-m gpu`).
Random inputs use numpy's PCG64 instead of libstdc++'s uniform_real_distribution
(not portable); tolerances and known answers are the reference's.
"""
import numpy as np
import pytest

from impls import B200Impl, OracleImpl, ShapeError, SingularMatrix, SingularSplit, pinv, rel_err, rel_fro

IMPLS = [pytest.param(OracleImpl(), id="oracle"), pytest.param(B200Impl(), id="b200", marks=pytest.mark.gpu)]


def rnd(seed, r, c):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(r, c))


def one_hot(rng, n, m):
    y = np.zeros((n, m))
    y[np.arange(n), rng.integers(0, m, size=n)] = 1.0
    return y


# ---------------------------------------------------------------- pinv_svd (test_linalg.cpp:26-58)
@pytest.mark.parametrize("impl", IMPLS)
def test_pinv_identity_and_rank_deficient_diagonal(impl):  # :26-32
    assert np.abs(impl.pinv_svd(np.eye(4)) - np.eye(4)).max() < 1e-12
    assert np.abs(impl.pinv_svd(np.array([[2.0, 0], [0, 0]])) - np.array([[0.5, 0], [0, 0]])).max() < 1e-14


@pytest.mark.parametrize("impl", IMPLS)
def test_pinv_left_inverse_full_column_rank(impl):  # :34-38
    a = rnd(11, 10, 4)
    assert np.abs(impl.pinv_svd(a) @ a - np.eye(4)).max() < 1e-10


@pytest.mark.parametrize("impl", IMPLS)
def test_pinv_penrose_conditions(impl):  # :40-58 (random shapes up to 50 x 50, half rank-deficient)
    rng = np.random.default_rng(12)
    for c in range(20):
        rows, cols = 2 + int(rng.integers(0, 49)), 2 + int(rng.integers(0, 49))
        a = rng.uniform(-1, 1, (rows, cols))
        if c % 2 == 0:
            a[:, cols - 1] = 2.0 * a[:, 0]
        x = impl.pinv_svd(a)
        assert rel_err(a @ x @ a, a) < 1e-8
        assert rel_err(x @ a @ x, x) < 1e-8
        assert rel_err(a @ x, (a @ x).T) < 1e-8
        assert rel_err(x @ a, (x @ a).T) < 1e-8


@pytest.mark.parametrize("impl", IMPLS)
def test_pinv_matches_numpy_svd_with_cut(impl):  # linalg.cpp:76-83 cut rule, incl. explicit tol
    rng = np.random.default_rng(21)
    for rows, cols, rank, tol in [(70, 33, 33, 0.0), (33, 70, 33, 0.0), (90, 45, 12, 0.0), (45, 90, 12, 0.0),
                                  (64, 64, 64, 1e-3), (130, 97, 60, 0.0)]:
        a = rng.uniform(-1, 1, (rows, rank)) @ rng.uniform(-1, 1, (rank, cols))
        if rank == min(rows, cols) and tol > 0:
            u, _, vt = np.linalg.svd(a, full_matrices=False)
            a = (u * np.logspace(0, -6, len(vt))) @ vt  # singular values straddle the explicit cut
        want = pinv(a, tol)
        assert rel_fro(impl.pinv_svd(a, tol), want) < 1e-9, (rows, cols, rank, tol)


# ---------------------------------------------------------------- matrix (test_matrix.cpp)
@pytest.mark.parametrize("impl", IMPLS)
def test_gram_equals_ata(impl):  # test_matrix.cpp:62-66 (1e-13)
    h = rnd(4, 9, 4)
    g = impl.gram(h)
    assert np.abs(g - h.T @ h).max() < 1e-13
    assert np.array_equal(g, g.T)  # lower triangle + mirror: exactly symmetric


@pytest.mark.parametrize("impl", IMPLS)
def test_gram_larger_and_odd_shapes(impl):
    for r, c in [(1, 1), (3, 7), (130, 129), (257, 200), (1000, 65)]:
        h = rnd(r * 7 + c, r, c)
        g = impl.gram(h)
        assert np.abs(g - h.T @ h).max() <= 1e-13 * max(1.0, r)
        assert np.array_equal(g, g.T)


# ---------------------------------------------------------------- linalg (test_linalg.cpp)
@pytest.mark.parametrize("impl", IMPLS)
def test_solve_spd_trivial_and_diagonal(impl):  # :60-68
    rhs = np.array([[8.0], [27.0]])
    assert np.abs(impl.solve_spd(np.eye(2), rhs) - rhs).max() < 1e-14
    x = impl.solve_spd(np.diag([4.0, 9.0]), rhs)
    assert x[0, 0] == pytest.approx(2.0, rel=1e-12)
    assert x[1, 0] == pytest.approx(3.0, rel=1e-12)


@pytest.mark.parametrize("impl", IMPLS)
def test_solve_spd_matches_pinv(impl):  # :70-76
    g = rnd(13, 6, 6)
    m = g.T @ g + np.eye(6)
    rhs = rnd(113, 6, 2)
    assert rel_err(impl.solve_spd(m, rhs), pinv(m) @ rhs) < 1e-8


@pytest.mark.parametrize("impl", IMPLS)
def test_solve_spd_reports_failing_pivot(impl):  # :78-90
    with pytest.raises(SingularMatrix) as e:
        impl.solve_spd(np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([[1.0], [1.0]]))
    assert e.value.pivot_index == 1
    assert abs(e.value.pivot_value) < 1e-12
    with pytest.raises(ValueError):
        impl.solve_spd(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[1.0], [1.0]]))
    with pytest.raises(ShapeError):
        impl.solve_spd(np.zeros((2, 3)), np.array([[1.0], [1.0]]))


@pytest.mark.parametrize("impl", IMPLS)
def test_rank_identity_and_engineered_dependency(impl):  # :92-116
    order, rank, _, _ = impl.rrf(np.eye(5))
    assert rank == 5 and sorted(order) == list(range(5))
    a = rnd(14, 6, 4)
    a[:, 2] = a[:, 0] + a[:, 1]
    order, rank, _, _ = impl.rrf(a, 1e-6)
    assert rank == 3
    basis = a[:, order[:3]]
    assert impl.rrf(basis, 1e-6)[1] == 3
    assert round(np.trace(pinv(a, 1e-6) @ a)) == 3


@pytest.mark.parametrize("impl", IMPLS)
def test_random_tall_matrices_full_rank(impl):  # :118-126
    rng = np.random.default_rng(15)
    for _ in range(10):
        cols = 3 + int(rng.integers(0, 8))
        rows = cols + int(rng.integers(0, 20))
        assert impl.rrf(rng.uniform(-1, 1, (rows, cols)))[1] == cols


@pytest.mark.parametrize("impl", IMPLS)
def test_zero_matrix_rank_zero_identity_order(impl):  # :128-132
    order, rank, _, _ = impl.rrf(np.zeros((4, 3)))
    assert rank == 0 and list(order) == [0, 1, 2]


@pytest.mark.parametrize("impl", IMPLS)
def test_rank_detection_deterministic(impl):  # :134-141
    a = rnd(16, 12, 7)
    r1, r2 = impl.rrf(a, 1e-9), impl.rrf(a, 1e-9)
    assert list(r1[0]) == list(r2[0]) and r1[1] == r2[1]


@pytest.mark.parametrize("impl", IMPLS)
def test_factor_reproduces_permuted_gram_and_solves(impl):  # :143-175
    a = rnd(18, 14, 6)
    order, rank, _, f = impl.rrf(a)
    assert rank == 6
    g = a.T @ a
    ffT = f @ f.T
    for i in range(6):
        for j in range(6):
            assert abs(ffT[i, j] - g[order[i], order[j]]) < 1e-10 * (1.0 + abs(g[i, j]))
    y = rnd(118, 14, 2)
    htyp = (a.T @ y)[order]
    beta = np.empty_like(htyp)
    beta[order] = impl.solve_factored_gram(f, order, rank, htyp)
    assert rel_err(beta, pinv(a) @ y) < 1e-8
    dep = rnd(218, 10, 4)
    dep[:, 3] = dep[:, 0]
    o2, r2, _, f2 = impl.rrf(dep, 1e-6)
    assert r2 == 3
    with pytest.raises(ValueError):
        impl.solve_factored_gram(f2, o2, r2, np.zeros((4, 1)))
    with pytest.raises(ShapeError):
        impl.solve_factored_gram(f, order, rank, np.zeros((3, 1)))


@pytest.mark.parametrize("impl", IMPLS)
def test_rank_tolerance_validation(impl):  # linalg.cpp:158-163
    with pytest.raises(ValueError):
        impl.rrf(rnd(1, 5, 3), -1.0)


# ---------------------------------------------------------------- elm (test_elm.cpp)
@pytest.mark.parametrize("impl", IMPLS)
def test_init_hidden_seed_deterministic_in_range(impl):  # :12-29
    w1, b1 = impl.init_hidden(4, 6, 2, 99)
    w2, b2 = impl.init_hidden(4, 6, 2, 99)
    w3, _ = impl.init_hidden(4, 6, 2, 100)
    assert np.array_equal(w1, w2) and np.array_equal(b1, b2)
    assert not np.array_equal(w1, w3)
    assert (w1 >= -1).all() and (w1 <= 1).all()


@pytest.mark.parametrize("impl", IMPLS)
def test_hidden_matrix_half_at_zero_preactivation(impl):  # :31-45
    h = impl.hidden_matrix(np.zeros((3, 4)), np.zeros((1, 4)), np.array([[0.3, -0.1, 0.9], [0.0, 0.5, -0.5]]))
    assert (h == 0.5).all()
    assert impl.hidden_matrix(np.array([[2.0]]), np.array([[-1.0]]), np.array([[0.5]]))[0, 0] == 0.5
    with pytest.raises(ShapeError):
        impl.hidden_matrix(np.zeros((3, 4)), np.zeros((1, 4)), np.zeros((2, 2)))


@pytest.mark.parametrize("impl", IMPLS)
def test_hidden_matrix_matches_scalar_loop(impl):  # :47-62 (1e-12)
    w, b = impl.init_hidden(5, 7, 1, 3)
    x = rnd(21, 9, 5)
    h = impl.hidden_matrix(w, b, x)
    z = x @ w + b
    assert np.abs(h - 1.0 / (1.0 + np.exp(-z))).max() < 1e-12
    assert (h > 0).all() and (h < 1).all()


@pytest.mark.parametrize("impl", IMPLS)
def test_solve_direct_trivial_systems(impl):  # :64-73
    y = rnd(22, 4, 2)
    beta, _ = impl.solve_beta(np.eye(4), y, "direct")
    assert rel_err(beta, y) < 1e-12
    beta, _ = impl.solve_beta(np.array([[1.0], [1.0]]), np.array([[1.0], [3.0]]), "direct")
    assert beta[0, 0] == pytest.approx(2.0, rel=1e-12)


@pytest.mark.parametrize("impl", IMPLS)
def test_solve_direct_matches_svd(impl):  # :75-80 (1e-8)
    h, y = rnd(23, 30, 8), rnd(123, 30, 2)
    assert rel_err(impl.solve_beta(h, y, "direct")[0], pinv(h) @ y) < 1e-8


@pytest.mark.parametrize("impl", IMPLS)
def test_df_split_equals_pinv_for_every_split(impl):  # :82-92 (block split == pinv, all splits)
    h, y = rnd(24, 25, 9), rnd(124, 25, 3)
    want = pinv(h) @ y
    for split in range(1, 9):
        assert rel_err(impl.solve_beta(h, y, "df", split)[0], want) < 1e-8


@pytest.mark.parametrize("impl", IMPLS)
def test_duplicate_column_ridge_or_fallback(impl):  # :102-118
    h1 = rnd(26, 12, 3)
    h = np.hstack([h1, h1[:, :1]])
    y = rnd(126, 12, 2)
    fitted_oracle = h @ (pinv(h) @ y)
    beta, diag = impl.solve_beta(h, y, "df", 3)
    assert diag["ridge_applied"] or diag["fallback_to_direct"]
    assert rel_err(h @ beta, fitted_oracle) < 1e-6


@pytest.mark.parametrize("impl", IMPLS)
def test_rank_path_engineered_dependent_column(impl):  # :120-133
    h = rnd(27, 30, 6)
    h[:, 4] = h[:, 1] - h[:, 3]
    y = rnd(127, 30, 2)
    beta, diag = impl.solve_beta(h, y, "rank", 0, 1e-6)
    assert diag["rank"] == 5 and diag["split_lo"] == 5 and diag["split_hi"] == 1
    assert rel_err(h @ beta, h @ (pinv(h) @ y)) < 1e-6


@pytest.mark.parametrize("impl", IMPLS)
def test_df_and_rank_predict_identically(impl):  # :135-155
    rng = np.random.default_rng(28)
    x = rng.uniform(-1, 1, (40, 5))
    y = one_hot(rng, 40, 3)
    b_df, _, w, b = impl.train(5, 10, 3, 7, x, y, "df", 4)
    b_rb, d_rb, _, _ = impl.train(5, 10, 3, 7, x, y, "rank")
    assert d_rb["rank"] == 10 and d_rb["split_lo"] == 5
    p_df, p_rb = impl.predict(w, b, b_df, x), impl.predict(w, b, b_rb, x)
    assert (p_df.argmax(1) == p_rb.argmax(1)).all()


@pytest.mark.parametrize("impl", IMPLS)
def test_consistent_targets_zero_residual(impl):  # :157-165
    w, b = impl.init_hidden(4, 8, 2, 11)
    x = rnd(29, 20, 4)
    h = impl.hidden_matrix(w, b, x)
    y = h @ rnd(129, 8, 2)
    beta, _, _, _ = impl.train(4, 8, 2, 11, x, y, "direct")
    assert np.linalg.norm(h @ beta - y) < 1e-8 * (1.0 + np.linalg.norm(y))


@pytest.mark.parametrize("impl", IMPLS)
def test_train_validates_shapes_and_n_ge_l(impl):  # :167-179
    rng = np.random.default_rng(30)
    x = rng.uniform(-1, 1, (6, 3))
    y = one_hot(rng, 6, 2)
    with pytest.raises(ValueError, match="direct"):
        impl.train(3, 10, 2, 1, x, y, "rank")
    with pytest.raises(ValueError):
        impl.train(3, 4, 2, 1, x, y, "df", 0)
    with pytest.raises(ValueError):
        impl.train(3, 4, 2, 1, x, y, "df", 4)
    with pytest.raises(ShapeError):
        impl.train(3, 4, 2, 1, x, np.zeros((5, 2)), "direct")


@pytest.mark.parametrize("impl", IMPLS)
def test_train_is_pure(impl):  # :181-189 (bitwise-equal beta)
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, (15, 4))
    y = one_hot(rng, 15, 2)
    b1 = impl.train(4, 6, 2, 5, x, y, "rank")[0]
    b2 = impl.train(4, 6, 2, 5, x, y, "rank")[0]
    assert np.array_equal(b1, b2)


@pytest.mark.parametrize("impl", IMPLS)
def test_residual_optimality_every_strategy(impl):  # :191-210
    rng = np.random.default_rng(32)
    for c in range(10):
        cols = 4 + int(rng.integers(0, 6))
        rows = cols + 5 + int(rng.integers(0, 30))
        h = rng.uniform(-1, 1, (rows, cols))
        if c % 2 == 0:
            h[:, cols - 1] = h[:, 0] + h[:, 1]
        y = rng.uniform(-1, 1, (rows, 2))
        best = np.linalg.norm(h @ (pinv(h) @ y) - y)
        for kind, split, tol in [("direct", 0, 0.0), ("df", cols // 2, 0.0), ("rank", 0, 1e-6)]:
            beta = impl.solve_beta(h, y, kind, split, tol)[0]
            assert np.linalg.norm(h @ beta - y) <= best + 1e-6 * (1.0 + np.linalg.norm(y))


@pytest.mark.parametrize("impl", IMPLS)
def test_accuracy_argmax_lowest_index_ties(impl):  # :212-220
    y = np.array([[1.0, 0], [0, 1], [1, 0]])
    assert impl.accuracy(y, y) == 1.0
    assert impl.accuracy(np.array([[0.0, 1], [1, 0], [0, 1]]), y) == 0.0
    assert impl.accuracy(np.array([[0.5, 0.5], [0.2, 0.8], [0.9, 0.1]]), y) == 1.0
    with pytest.raises(ShapeError):
        impl.accuracy(y, np.zeros((2, 2)))


# ---------------------------------------------------------------- acceptance.cpp / checks.cpp
@pytest.mark.parametrize("impl", IMPLS)
def test_acceptance_c1_block_and_rank_equal_pinv(impl):  # acceptance.cpp:52-74 (subset of the 200)
    rng = np.random.default_rng(1001)
    worst = 0.0
    for _ in range(25):
        L = 4 + int(rng.integers(0, 47))
        n = max(20, L) + int(rng.integers(0, 150))
        m = 1 + int(rng.integers(0, 5))
        h = rng.uniform(-1, 1, (n, L))
        y = rng.uniform(-1, 1, (n, m))
        want = pinv(h) @ y
        for split in sorted({1, L // 2, L - 1}):
            worst = max(worst, rel_err(impl.solve_beta(h, y, "df", split)[0], want))
        worst = max(worst, rel_err(impl.solve_beta(h, y, "rank")[0], want))
    assert worst < 1e-6


@pytest.mark.parametrize("impl", IMPLS)
def test_acceptance_c2_rank_deficient_fitted_values(impl):  # acceptance.cpp:78-108
    rng = np.random.default_rng(1002)
    worst = 0.0
    for _ in range(50):
        L = 6 + int(rng.integers(0, 15))
        n = L + 10 + int(rng.integers(0, 60))
        defi = 1 + int(rng.integers(0, 2))
        h = rng.uniform(-1, 1, (n, L))
        for dd in range(defi):
            s1, s2 = int(rng.integers(0, L - defi)), int(rng.integers(0, L - defi))
            h[:, L - 1 - dd] = h[:, s1] + 0.5 * h[:, s2]
        y = rng.uniform(-1, 1, (n, 2))
        beta, diag = impl.solve_beta(h, y, "rank", 0, 1e-6)
        assert diag["rank_known"] and diag["rank"] < L
        fo = h @ (pinv(h) @ y)
        worst = max(worst, np.linalg.norm(h @ beta - fo) / (1.0 + np.linalg.norm(fo)))
    assert worst < 1e-6


@pytest.mark.parametrize("impl", IMPLS)
def test_acceptance_c7_degenerate_inputs(impl):  # acceptance.cpp:233-281
    beta, diag = impl.solve_beta(np.zeros((10, 4)), np.ones((10, 2)), "rank")
    assert diag["rank"] == 0 and diag["fallback_to_direct"] and np.abs(beta).max() == 0.0
    # constant (normalised-to-zero) features still train to a finite beta
    y = np.zeros((20, 2))
    y[np.arange(20), np.arange(20) % 2] = 1.0
    beta, _, _, _ = impl.train(3, 5, 2, 1, np.zeros((20, 3)), y, "rank")
    assert np.isfinite(beta).all()
    # single-class targets: training accuracy 1.0
    rng = np.random.default_rng(3)
    _, diag, _, _ = impl.train(4, 6, 1, 2, rng.uniform(0, 1, (25, 4)), np.ones((25, 1)), "rank")
    assert diag["training_accuracy"] == 1.0


@pytest.mark.parametrize("impl", IMPLS)
def test_checks_rank_matches_svd_count(impl):  # checks.cpp:136-152 (rank vs SVD count at 1e-6)
    rng = np.random.default_rng(77)
    for c in range(20):
        rows = 12 + int(rng.integers(0, 40))
        cols = min(2 + int(rng.integers(0, 10)), rows - 2)
        a = rng.uniform(-1, 1, (rows, cols))
        if c % 3 == 0 and cols >= 2:
            a[:, cols - 1] = a[:, 0] + a[:, 1 % cols]
        assert impl.rrf(a, 1e-6)[1] == round(np.trace(pinv(a, 1e-6) @ a))
