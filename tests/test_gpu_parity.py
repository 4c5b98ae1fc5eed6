"""GPU parity on BASELINE.json's configs: the B200 path (C ABI -> sm_100a kernels)
against the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star):
  * rank, pivot order and predicted labels bit-exact (C3: pivots modulo exact-twin classes);
  * beta within relative Frobenius max(1e-9, 4 * oracle self-floor), the floor being the
    oracle's own 1-vs-8-row-shard Gram summation difference;
  * H within 1e-12 elementwise (reference test_elm.cpp:75);
  * configs beyond the oracle's reach are checked through size-independent properties
    (pivots of the oracle factorisation applied to the GPU's own Gram, FF^T = P^T G P,
    normal-equation backward error, accuracy re-derived from predictions).
"""
import numpy as np
import pytest

import oracle
import paper_2011_02436_b200 as rb

pytestmark = pytest.mark.gpu

SEED_X, SEED_T, SEED_W = 1001, 2001, 3001


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def self_floor(h, t, tol=0.0):
    b1, _, _ = oracle.solve_beta(h, t, "rank", 0, tol, 1)
    b8, _, _ = oracle.solve_beta(h, t, "rank", 0, tol, 8)
    return rel_fro(b8, b1)


def top2_gap(scores):
    """Min over rows of (best - runner-up) score: how close the arg-max labels are to flipping."""
    s = np.sort(np.asarray(scores), axis=1)
    return float((s[:, -1] - s[:, -2]).min()) if s.shape[1] > 1 else float("inf")


def floor_from_grams(h, t, L, m, n):
    """Oracle self-floor without an extra train(): beta from the 1-shard and the 8-shard augmented
    Gram [H T]^T [H T] (the H^T T block sums products in the same row order as matmul_at), each
    factored and solved by the oracle.  Returns (floor, beta_1shard, order_1shard)."""
    out = []
    for shards in (1, 8):
        ga = oracle.gram(np.hstack([h, t]), shards)
        order, rank, _, f, _ = oracle.factor_gram(np.ascontiguousarray(ga[:L, :L]), n)
        xs = oracle.solve_factored_gram(f, order, rank, ga[:L, L:L + m][order])
        beta = np.empty_like(xs)
        beta[order] = xs
        out.append((beta, order))
    return rel_fro(out[1][0], out[0][0]), out[0][0], out[0][1]


def train_both(n, d, L, m, seeds=(SEED_X, SEED_T, SEED_W), tol=0.0):
    x, t = rb.synth_classification(n, d, m, seeds[0], seeds[1])
    params = rb.ElmParams(d, L, m, seeds[2])
    model, diag, order = rb.train(params, x, t, rb.SolverStrategy.rank_based(tol), return_order=True)
    ref = oracle.train(d, L, m, seeds[2], x, t, "rank", 0, tol)
    return x, t, model, diag, order, ref


@pytest.mark.parametrize("cfg", [
    pytest.param((2000, 16, 200, 2), id="C1"),
    pytest.param((50000, 64, 1000, 10), id="C2"),
])
def test_train_parity_baseline_configs(cfg):
    n, d, L, m = cfg
    x, t, model, diag, order, ref = train_both(n, d, L, m)
    assert diag.rank == ref["diag"]["rank"] == L
    assert order == ref["order"], "pivot order differs from the oracle"
    assert np.array_equal(model.hidden.weights, ref["w"]) and np.array_equal(model.hidden.biases, ref["b"])
    h_o = oracle.hidden_matrix(ref["w"], ref["b"], x)
    floor = self_floor(h_o, t)
    tol = max(1e-9, 4 * floor)
    err = rel_fro(model.beta, ref["beta"])
    print(f"{cfg}: beta rel {err:.3e} (floor {floor:.3e}, gate {tol:.1e}), margin {ref['diag']['min_pivot_margin']:.2e}")
    assert err <= tol
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]
    assert diag.split_lo == (L + 1) // 2 and diag.split_hi == L // 2 and not diag.fallback_to_direct
    # predicted labels on the training rows and on 1000 seeded test rows
    xt, _ = rb.synth_classification(1000, d, m, SEED_X + 100, SEED_T)
    for xx in (x, xt):
        s = rb.predict(model, xx)
        so = oracle.predict(ref["w"], ref["b"], ref["beta"], xx)
        assert (s.argmax(1) == so.argmax(1)).all()
        assert rel_fro(s, so) < 1e-8
        print(f"  min top-2 logit gap {top2_gap(so):.3e} over {len(so)} rows")


def test_hidden_matrix_parity_c1():
    x, _ = rb.synth_classification(2000, 16, 2, SEED_X, SEED_T)
    hid = rb.init_hidden(rb.ElmParams(16, 200, 2, SEED_W))
    h = rb.hidden_matrix(hid, x)
    ho = oracle.hidden_matrix(hid.weights, hid.biases, x)
    assert np.abs(h - ho).max() < 1e-12


@pytest.mark.parametrize("shape", [(5, 3, 1, 1), (40, 5, 10, 3), (129, 7, 65, 3), (300, 33, 129, 5),
                                   (1000, 17, 257, 7), (4097, 130, 300, 1), (700, 3, 64, 2),
                                   # m = 32 / 33: the augmented-factorisation boundary (forward sweep
                                   # inside the panels vs. the two-sweep TRSM)
                                   (3000, 20, 200, 32), (3000, 20, 200, 33),
                                   # L + m = 1025: the first panel on the shared-memory cluster variant
                                   (6000, 40, 1015, 10), (8000, 30, 1200, 4)])
def test_train_parity_ragged_shapes(shape):
    n, d, L, m = shape
    x, t, model, diag, order, ref = train_both(n, d, L, m, seeds=(n, d + 1, L + 2))
    assert diag.rank == ref["diag"]["rank"]
    assert diag.fallback_to_direct == bool(ref["diag"]["fallback_to_direct"])
    if L >= 2:
        assert order == ref["order"]
    h = oracle.hidden_matrix(ref["w"], ref["b"], x)
    if diag.rank == L:  # gate on the oracle's own reduction-order floor (ill-conditioned small-d cases)
        assert rel_fro(model.beta, ref["beta"]) <= max(1e-8, 4 * self_floor(h, t))
    else:  # beta is non-unique when rank < L: compare fitted values
        assert rel_fro(h @ model.beta, h @ ref["beta"]) < 1e-8
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]


def test_determinism_bitwise():
    x, t = rb.synth_classification(3000, 20, 4, 5, 6)
    p = rb.ElmParams(20, 300, 4, 7)
    b1 = rb.train(p, x, t, rb.SolverStrategy.rank_based())[0].beta
    b2 = rb.train(p, x, t, rb.SolverStrategy.rank_based())[0].beta
    assert np.array_equal(b1, b2)


def twin_classes(L, tgt, src):
    cls = np.arange(L)
    for a, b in zip(tgt, src):
        cls[a] = b
    return cls


def test_c3_rank_deficient_twins():
    """C3: N=20000, d=32 (16 base + 16 linear combinations), L=2000 with 500 exact duplicate nodes,
    m=5; hidden_matrix + solve_beta(rank_based(1e-6)) as SURVEY §8(b) prescribes."""
    n, base, L, m = 20000, 16, 2000, 5
    x, t = rb.synth_rank_deficient(n, base, m, SEED_X, 4001, SEED_T)
    hid0 = rb.init_hidden(rb.ElmParams(2 * base, L, m, SEED_W))
    hid, tgt, src = rb.duplicate_nodes(hid0, 500, 5001)
    cls = twin_classes(L, tgt, src)
    h = rb.hidden_matrix(hid, x)
    ho = oracle.hidden_matrix(hid.weights, hid.biases, x)
    assert np.array_equal(h[:, tgt], h[:, src]) and np.array_equal(ho[:, tgt], ho[:, src])  # exact twins
    diag = rb.SolveDiagnostics()
    beta = rb.solve_beta(h, t, rb.SolverStrategy.rank_based(1e-6), diag)
    beta_o, diag_o, order_o = oracle.solve_beta(ho, t, "rank", 0, 1e-6)
    assert diag.rank == diag_o["rank"] == 1500
    assert diag.ridge_applied == bool(diag_o["ridge_applied"])
    assert diag.fallback_to_direct == bool(diag_o["fallback_to_direct"])
    f = rb.rank_revealing_factor(h, 1e-6)
    assert f.permutation.rank == 1500
    order = f.permutation.order
    r = 1500
    assert [cls[i] for i in order[:r]] == [cls[i] for i in order_o[:r]], "pivots differ beyond twin classes"
    print("raw pivot order identical:", order[:r] == order_o[:r])
    fit, fit_o = h @ beta, ho @ beta_o
    err = rel_fro(fit, fit_o)
    print(f"C3 fitted rel {err:.3e}, beta rel {rel_fro(beta, beta_o):.3e} (beta is non-unique)")
    assert err < 1e-8
    assert (fit.argmax(1) == fit_o.argmax(1)).all()


def test_c3_small_duplicates():
    n, d, L, m = 3000, 12, 200, 3
    x, t = rb.synth_classification(n, d, m, 31, 32)
    hid, tgt, src = rb.duplicate_nodes(rb.init_hidden(rb.ElmParams(d, L, m, 33)), 40, 34)
    cls = twin_classes(L, tgt, src)
    h = rb.hidden_matrix(hid, x)
    ho = oracle.hidden_matrix(hid.weights, hid.biases, x)
    diag = rb.SolveDiagnostics()
    beta = rb.solve_beta(h, t, rb.SolverStrategy.rank_based(1e-6), diag)
    beta_o, diag_o, order_o = oracle.solve_beta(ho, t, "rank", 0, 1e-6)
    assert diag.rank == diag_o["rank"] == L - 40
    order = rb.rank_revealing_factor(h, 1e-6).permutation.order
    assert [cls[i] for i in order[:L - 40]] == [cls[i] for i in order_o[:L - 40]]
    assert rel_fro(h @ beta, ho @ beta_o) < 1e-8


def _device_stages(n, d, L, m, seeds, tol=0.0):
    import torch

    x, t = rb.synth_classification(n, d, m, seeds[0], seeds[1])
    hid = rb.init_hidden(rb.ElmParams(d, L, m, seeds[2]))
    X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    G = torch.empty((L, L), dtype=torch.float64, device="cuda")
    HtT = torch.empty((L, m), dtype=torch.float64, device="cuda")
    rb.gram_stage_device(X, T, W, B, G, HtT)
    beta, diag, order = rb.solve_stage_device(G, HtT, n, rb.SolverStrategy.rank_based(tol), return_order=True)
    hits = rb.accuracy_stage_device(X, T, W, B, beta)
    return x, t, hid, G.cpu().numpy(), HtT.cpu().numpy(), beta.cpu().numpy(), diag, order, hits


@pytest.mark.parametrize("L", [250, 500, 1000, 2000, 4000, pytest.param(8000, marks=pytest.mark.slow)])
def test_c4_sweep_vs_oracle(L):
    """BASELINE config 4 (N=100000, d=128, m=10) end to end at every L of the sweep: the GPU train()
    against the oracle's train() on the same seeded inputs.  Rank, the whole pivot order and the
    training accuracy bit-exact; beta within max(1e-9, 4 x the oracle's 1-vs-8-shard floor); labels
    of 20000 training rows bit-exact.  L = 8000 runs the >4096-label grid panel for its first panels."""
    n, d, m = 100000, 128, 10
    x, t, model, diag, order, ref = train_both(n, d, L, m, seeds=(SEED_X + 4, SEED_T + 4, SEED_W + L))
    assert diag.rank == ref["diag"]["rank"] == L
    assert order == ref["order"], "pivot order differs from the oracle"
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]
    h = oracle.hidden_matrix(ref["w"], ref["b"], x)
    floor, beta1, order1 = floor_from_grams(h, t, L, m, n)
    assert order1 == ref["order"]
    assert np.array_equal(beta1, ref["beta"])  # augmented-Gram H^T T == matmul_at, bitwise
    err = rel_fro(model.beta, ref["beta"])
    gate = max(1e-9, 4 * floor)
    so = oracle.predict(ref["w"], ref["b"], ref["beta"], x[:20000])
    s = rb.predict(model, x[:20000])
    print(f"C4 L={L}: beta rel {err:.3e} (floor {floor:.3e}, gate {gate:.1e}), margin "
          f"{ref['diag']['min_pivot_margin']:.2e}, min top-2 gap {top2_gap(so):.2e}")
    assert err <= gate
    assert (s.argmax(1) == so.argmax(1)).all()


def _pivots_on_device_gram(n, d, L, m, seeds, tol=0.0):
    """Device Gram and solve (stage API), then the oracle's factorisation of the SAME Gram."""
    x, t, hid, G, HtT, beta, diag, order, hits = _device_stages(n, d, L, m, seeds, tol)
    assert np.array_equal(G, G.T)
    o_ord, o_rank, _, o_f, margin = oracle.factor_gram(G, n, tol)
    return x, t, hid, G, HtT, beta, diag, order, hits, o_ord, o_rank, o_f, margin


def test_c5_standin_pivots_vs_oracle():
    """C5 stand-in on one GPU (N reduced to 120k, d=256, L=8192, m=100): the device factorisation of
    the device Gram (the first 64 panels on the >4096-label grid panel) against the oracle's
    factorisation of the same Gram: rank and the whole pivot order bit-exact, beta against the
    oracle's solve on that Gram, normal-equation backward error."""
    n, d, L, m = 120000, 256, 8192, 100
    (x, t, hid, G, HtT, beta, diag, order, hits, o_ord, o_rank, o_f,
     margin) = _pivots_on_device_gram(n, d, L, m, (SEED_X + 5, SEED_T + 5, SEED_W + 5))
    assert diag.rank == o_rank == L
    assert list(order) == o_ord, "pivots differ from the oracle on the same Gram"
    bo = oracle.solve_factored_gram(o_f, o_ord, L, HtT[o_ord])
    beta_o = np.empty_like(bo)
    beta_o[o_ord] = bo
    bwd = np.linalg.norm(G @ beta - HtT) / (np.linalg.norm(G) * np.linalg.norm(beta))
    print(f"C5 stand-in: beta vs oracle-on-same-Gram {rel_fro(beta, beta_o):.3e}, margin {margin:.2e}, "
          f"backward error {bwd:.3e}, accuracy {hits / n:.4f}")
    assert rel_fro(beta, beta_o) < 1e-6  # C5 floor ~1e-6
    assert bwd < 1e-12


@pytest.mark.parametrize("L,ndup", [(5000, 0), (6000, 400), (9000, 300)])
def test_grid_panel_rank_deficient(L, ndup):
    """Rank stop inside a wide panel: d = 2 features make H numerically low-rank, so at tol 1e-6 the
    factorisation stops after a few dozen pivots with > 4096 labels live -- in the 32-wide 512-thread
    cluster panel (4096 < labels <= 8192) or, at L = 9000, the cooperative-grid panel (> 8192); with
    duplicated nodes the stop rule and the final swap also see exact twins.  Rank and pivots equal
    the oracle's factorisation of the device's own Gram (modulo twin classes); the rank-deficient
    solve (Schur block path) fits like the oracle's."""
    import torch

    n, d, m = 20000, 2, 3
    x, t = rb.synth_classification(n, d, m, 71, 72)
    hid0 = rb.init_hidden(rb.ElmParams(d, L, m, 73))
    hid, tgt, src = (hid0, [], []) if ndup == 0 else rb.duplicate_nodes(hid0, ndup, 74)
    cls = twin_classes(L, tgt, src)
    X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    G = torch.empty((L, L), dtype=torch.float64, device="cuda")
    HtT = torch.empty((L, m), dtype=torch.float64, device="cuda")
    rb.gram_stage_device(X, T, W, B, G, HtT)
    beta, diag, order = rb.solve_stage_device(G, HtT, n, rb.SolverStrategy.rank_based(1e-6), return_order=True)
    g = G.cpu().numpy()
    o_ord, o_rank, _, _, margin = oracle.factor_gram(g, n, 1e-6)
    r = diag.rank
    print(f"grid-panel stop: L={L} ndup={ndup} rank {r} (oracle {o_rank}), labels live at the stop {L - r}, "
          f"margin {margin:.2e}")
    assert r == o_rank and L - r > 4096
    assert [cls[i] for i in order[:r]] == [cls[i] for i in o_ord[:r]]
    h = oracle.hidden_matrix(hid.weights, hid.biases, x)
    beta_o, diag_o, _ = oracle.solve_beta(h, t, "rank", 0, 1e-6)
    assert diag_o["rank"] == r
    # rank ~22 of >= 5000 columns: the Schur block path (elm.cpp:124-156) solves a ~5000-wide block
    # of numerical rank ~0 after its ridge rescue (condition ~1e10), so individual fitted values
    # depend on Gram rounding at ~1e-4 (the oracle builds the blocks from H, the device from Gram
    # sub-blocks).  Both are solutions of the same regularised problem: the training residual and
    # the predicted labels must agree.
    fit, fit_o = h @ beta.cpu().numpy(), h @ beta_o
    res, res_o = np.linalg.norm(t - fit), np.linalg.norm(t - fit_o)
    agree = float((fit.argmax(1) == fit_o.argmax(1)).mean())
    print(f"  fitted rel {rel_fro(fit, fit_o):.3e}, residual {res:.9e} vs oracle {res_o:.9e}, labels agree "
          f"{agree:.5f}; ridge {diag.ridge_applied} / {diag_o['ridge_applied']}")
    assert diag.ridge_applied == bool(diag_o["ridge_applied"])
    # the device's Gram (exact int8 digit products) is closer to the exact H^T H than the oracle's
    # sequential sums: its regularised fit may be better, never worse beyond 1e-6, and the two
    # residuals agree to 1e-5 (measured: 39.662452 device vs 39.662497 oracle at L = 6000, ndup = 400)
    assert res <= res_o * (1 + 1e-6)
    assert abs(res - res_o) <= 1e-5 * res_o
    assert agree >= 0.999


def test_sharded_stages_equal_single_pass():
    """Two row shards on one GPU (the per-rank stages + a summed Gram, as the NCCL all-reduce does)."""
    import torch

    n, d, L, m = 30000, 32, 600, 6
    x, t = rb.synth_classification(n, d, m, 41, 42)
    params = rb.ElmParams(d, L, m, 43)
    hid = rb.init_hidden(params)
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    parts = []
    for r0, r1 in [(0, 17001), (17001, n)]:
        X, T = torch.from_numpy(x[r0:r1]).cuda(), torch.from_numpy(t[r0:r1]).cuda()
        G = torch.empty((L, L), dtype=torch.float64, device="cuda")
        HtT = torch.empty((L, m), dtype=torch.float64, device="cuda")
        rb.gram_stage_device(X, T, W, B, G, HtT, keep_h=False)
        parts.append((G, HtT, X, T))
    G = parts[0][0] + parts[1][0]
    HtT = parts[0][1] + parts[1][1]
    beta, diag, order = rb.solve_stage_device(G, HtT, n, rb.SolverStrategy.rank_based(), return_order=True)
    hits = sum(rb.accuracy_stage_device(X, T, W, B, beta) for _, _, X, T in parts)
    model, d1, order1 = rb.train(params, x, t, rb.SolverStrategy.rank_based(), return_order=True)
    assert order == order1 and diag.rank == d1.rank == L
    assert rel_fro(beta.cpu().numpy(), model.beta) < 1e-9
    assert hits / n == d1.training_accuracy


def test_errors_from_device_path():
    with pytest.raises(rb.SingularMatrix) as e:
        rb.solve_spd(np.diag([1.0, 0.0, 2.0]), np.ones((3, 1)))
    assert e.value.pivot_index == 1
    with pytest.raises(ValueError, match="direct"):
        rb.train(rb.ElmParams(3, 50, 2, 1), np.zeros((10, 3)), np.zeros((10, 2)), rb.SolverStrategy.rank_based())
    with pytest.raises(ValueError):
        rb.rank_revealing_factor(np.ones((4, 2)), -1.0)
    with pytest.raises(rb.ShapeError):
        rb.hidden_matrix(rb.init_hidden(rb.ElmParams(3, 4, 1, 1)), np.zeros((2, 5)))


@pytest.mark.parametrize("n,m", [(200, 2), (256, 1), (257, 3), (1000, 10), (2047, 130), (4100, 100)])
def test_triangular_solve_pair_sizes(n, m):
    """K4 on its own: (F F^T)^-1 rhs for many block counts / CTA counts / RHS chunks."""
    rng = np.random.default_rng(n + m)
    f = np.tril(rng.uniform(-0.1, 0.1, (n, n))) + np.eye(n) * 2.0
    rhs = rng.uniform(-1, 1, (n, m))
    perm = rb.ColumnPermutation(list(range(n)), n, 0.0)
    x = rb.solve_factored_gram(rb.RankRevealingFactor(perm, f), rhs)
    assert rel_fro(x, np.linalg.solve(f @ f.T, rhs)) < 1e-13


def test_augmented_stage_api_row_shards():
    """Row-sharded augmented stages on one device (the multi-GPU path without NCCL): three row
    blocks accumulate [H T]^T [H T] in one buffer, one solve on it.  Pivots, rank and accuracy equal
    the unsharded train(); beta within the reduction-order floor."""
    import torch

    n, d, L, m = 30000, 48, 600, 6
    x, t = rb.synth_classification(n, d, m, 11, 12)
    params = rb.ElmParams(d, L, m, 13)
    hid = rb.init_hidden(params)
    model, diag0, order0 = rb.train(params, x, t, rb.SolverStrategy.rank_based(), return_order=True)
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    gaug = torch.empty((L + m, L + m), dtype=torch.float64, device="cuda")
    hits = 0
    bounds = [(0, 9000), (9000, 21111), (21111, n)]
    for i, (a, b) in enumerate(bounds):
        X = torch.from_numpy(np.ascontiguousarray(x[a:b])).cuda()
        T = torch.from_numpy(np.ascontiguousarray(t[a:b])).cuda()
        rb.gram_stage_device_aug(X, T, W, B, gaug, accumulate=i > 0, keep_h=False)
    beta, diag, order = rb.solve_stage_device_aug(gaug, L, m, n, rb.SolverStrategy.rank_based(), return_order=True)
    for a, b in bounds:
        X = torch.from_numpy(np.ascontiguousarray(x[a:b])).cuda()
        T = torch.from_numpy(np.ascontiguousarray(t[a:b])).cuda()
        hits += rb.accuracy_stage_device(X, T, W, B, beta)
    assert diag.rank == diag0.rank == L and order == order0
    assert hits / n == diag0.training_accuracy
    assert rel_fro(beta.cpu().numpy(), model.beta) < 1e-9


@pytest.mark.parametrize("kind,split", [("direct", 0), ("df", 400), ("df", 1)])
def test_other_strategies_at_scale(kind, split):
    """direct (unpivoted SpdFactor panels, elm.cpp:108-122) and df splits (Schur block path on Gram
    sub-blocks, elm.cpp:124-185) at N = 20000, L = 800 against the oracle."""
    n, d, L, m = 20000, 32, 800, 5
    x, t = rb.synth_classification(n, d, m, 41, 42)
    params = rb.ElmParams(d, L, m, 43)
    strat = rb.SolverStrategy.direct() if kind == "direct" else rb.SolverStrategy.df_split(split)
    model, diag = rb.train(params, x, t, strat)
    ref = oracle.train(d, L, m, 43, x, t, kind, split, 0.0)
    h = oracle.hidden_matrix(ref["w"], ref["b"], x)
    for k in ("ridge_applied", "fallback_to_direct", "used_svd_path"):
        assert getattr(diag, k) == bool(ref["diag"][k]), k
    floor = rel_fro(h @ (np.linalg.pinv(h) @ t), h @ ref["beta"])
    err = rel_fro(h @ model.beta, h @ ref["beta"])
    print(f"{kind}:{split}: fitted rel {err:.2e} (floor {floor:.2e}), beta rel {rel_fro(model.beta, ref['beta']):.2e}")
    assert err <= max(1e-9, 4 * floor)
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]
