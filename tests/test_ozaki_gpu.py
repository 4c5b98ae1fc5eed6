"""The train path's Gram on the INT8 tensor cores (csrc/k_ozaki.cu, rbpg_gram_int8_device): every fp64
column becomes 54-bit integers in 7 balanced int8 digit planes, 28 exact int8 products are summed in
int32 and combined in fp64.  Checked against an extended-precision (long double) Gram of the same
matrix: |G - exact| <= 4e-16 sqrt(G_aa G_bb) -- below a plain fp64 dot product's own error -- with
exact symmetry and bit-equal entries for identical columns (the C3 twin ties).  The reference's Gram
is linalg.cpp:179-184 (lower triangle of H^T H, mirrored)."""
import numpy as np
import pytest

import paper_2011_02436_b200 as rb

pytestmark = pytest.mark.gpu


def exact_gram(a):
    al = a.astype(np.longdouble)
    return al.T @ al


def tricky(n, m, seed):
    rng = np.random.default_rng(seed)
    a = 1.0 / (1.0 + np.exp(-(rng.uniform(-6, 6, (n, m)) + rng.normal(0, 3, m))))  # sigmoid columns
    a[:, 0] = 0.0                                       # all-zero column
    if m > 3:
        a[:, 3] = a[:, 1]                               # exact twin
        a[:, 2] = -a[:, 2] * 1e-3                       # negative, small scale
    if m > 6:
        a[:, 4] = (np.arange(n) % 3 == 0)               # one-hot target column
        a[:, 5] = a[:, 5] * np.where(np.arange(n) % 7 == 0, 1.0, 1e-9)  # wide dynamic range in a column
        a[:, 6] = rng.normal(0, 1, n) * 1e5             # signed, large
    return a


@pytest.mark.parametrize("n,m", [(777, 129), (5000, 300), (40000, 40), (3, 1), (1000, 7)])
def test_int8_gram_vs_exact(n, m):
    import torch

    a = tricky(n, m, n + m)
    A = torch.from_numpy(a).cuda()
    G = torch.full((m, m), np.nan, dtype=torch.float64, device="cuda")
    rb.gram_int8_device(A, G)
    g = G.cpu().numpy()
    ge = exact_gram(a)
    d = np.sqrt(np.maximum(np.diag(ge), 0))
    scale = np.outer(d, d)
    scale[scale == 0] = 1
    err = float((np.abs(g.astype(np.longdouble) - ge) / scale).max())
    seq = float((np.abs((a.T @ a).astype(np.longdouble) - ge) / scale).max())  # BLAS fp64 Gram, for scale
    print(f"n={n} m={m}: int8 Gram max err {err:.3e} of sqrt(Gaa Gbb) (fp64 BLAS Gram: {seq:.3e})")
    assert np.array_equal(g, g.T)
    assert err <= 4e-16
    if m > 3:
        assert np.array_equal(g[:, 1], g[:, 3]) and g[1, 1] == g[3, 3] == g[1, 3]
        assert (g[0] == 0).all()


def test_int8_gram_accumulate_and_leading_dims():
    import torch

    a = tricky(3000, 70, 5)
    big = torch.zeros((3000, 75), dtype=torch.float64, device="cuda")
    big[:, :70] = torch.from_numpy(a)
    G = torch.zeros((70, 72), dtype=torch.float64, device="cuda")
    G[:, :70] = torch.eye(70, dtype=torch.float64)
    rb.gram_int8_device(big[:, :70], G[:, :70], accumulate=True)
    ge = exact_gram(a) + np.eye(70)
    d = np.sqrt(np.diag(ge))
    err = float((np.abs(G[:, :70].cpu().numpy() - ge) / np.outer(d, d)).max())
    assert err <= 4e-16
    assert (G[:, 70:] == 0).all()


def test_int8_gram_matches_dmma_gram():
    """On a hidden layer the INT8 Gram is at least as accurate as the FP64 DMMA Gram."""
    import torch

    x, t = rb.synth_classification(20000, 64, 10, 11, 12)
    hid = rb.init_hidden(rb.ElmParams(64, 500, 10, 13))
    import oracle
    h = np.hstack([oracle.hidden_matrix(hid.weights, hid.biases, x), t])
    H = torch.from_numpy(h).cuda()
    g8 = torch.empty((510, 510), dtype=torch.float64, device="cuda")
    g64 = torch.empty_like(g8)
    rb.gram_int8_device(H, g8)
    rb.gram_device(H, g64)
    ge = exact_gram(h)
    d = np.sqrt(np.diag(ge))
    s = np.outer(d, d)
    s[s == 0] = 1  # empty classes: zero target columns
    e8 = float((np.abs(g8.cpu().numpy() - ge) / s).max())
    e64 = float((np.abs(g64.cpu().numpy() - ge) / s).max())
    print(f"hidden layer 20000 x 510: int8 Gram err {e8:.3e}, DMMA Gram err {e64:.3e}")
    # heavy-tailed sigmoid columns (max / rms ~ 30): the digit-plane error scales with max_a max_b / sqrt(N)
    # (dropped w >= 9 digit products), a blocked fp64 sum's with the rms -- measured 8.5e-16 vs 9.3e-16
    assert e8 <= 1e-15 and e8 <= e64 + 1e-17


@pytest.mark.parametrize("n,d,L", [(2000, 16, 200), (1000, 33, 129), (3000, 256, 300), (257, 64, 1), (5, 3, 7),
                                   (600, 130, 513)])
def test_int8_hidden_vs_extended_precision(n, d, L):
    """K1i (oz_hidden_kernel): H = sigmoid(X W + b) from 28 exact int8 digit-plane products, checked against
    the same formula in long double (elm.cpp:93-106: bias after the full dot product) and against the
    oracle's fp64 restatement."""
    import oracle

    x, _ = rb.synth_classification(n, d, 2, n + d, L + 1)
    x[:, 0] *= -3.0e-7                                    # a small, negative feature column
    hid = rb.init_hidden(rb.ElmParams(d, L, 2, n + L))
    h = rb.hidden_matrix(hid, x)
    xl, wl, bl = (a.astype(np.longdouble) for a in (x, hid.weights, hid.biases.reshape(1, -1)))
    z = xl @ wl + bl
    ref = 1.0 / (1.0 + np.exp(-z))
    err = float(np.abs(h.astype(np.longdouble) - ref).max())
    ho = oracle.hidden_matrix(hid.weights, hid.biases, x)
    err_o = float(np.abs(ho.astype(np.longdouble) - ref).max())
    print(f"n={n} d={d} L={L}: int8 H max err {err:.2e} (oracle fp64: {err_o:.2e})")
    assert err <= max(4e-16, 2.0 * err_o)
    assert np.abs(h - ho).max() < 1e-12


@pytest.mark.parametrize("n,d,L", [(1000, 32, 300), (4096, 64, 256), (77, 9, 40)])
def test_int8_hidden_saturating_and_partial_blocks(n, d, L):
    """K1i epilogue: blocks whose |z| exceeds 700 leave the in-range sigmoid and are recomputed with the
    full select chain (overflow to inf -> h = 0 exactly, underflow -> h = 1 exactly), as are the last,
    partial row blocks; blocks mixing both ranges must still equal the reference formula."""
    import oracle

    rng = np.random.default_rng(n + L)
    x = rng.random((n, d))
    scale = np.where(rng.random(n) < 0.5, 1.0, 180.0)     # half the rows drive |z| into the hundreds / thousands
    scale[::97] = 4000.0                                  # some far beyond the exp range: exact 0 / 1
    x *= scale[:, None]
    hid = rb.init_hidden(rb.ElmParams(d, L, 2, n + L))
    h = rb.hidden_matrix(hid, x)
    ho = oracle.hidden_matrix(hid.weights, hid.biases, x)
    z = x @ hid.weights + hid.biases.reshape(1, -1)
    assert np.isfinite(h).all() and (np.abs(z) > 745.2).any() and (np.abs(z) < 700).any()
    assert np.abs(h - ho).max() < 1e-12
    sat = np.abs(z) > 760
    assert np.array_equal(h[sat], ho[sat])                # exact 0.0 / 1.0 where the exponential saturates
    big = np.abs(z) > 40                                  # 1 ulp of e^-z relative to 1: h rounds like the oracle's
    assert np.abs(h[big] - ho[big]).max() <= 1e-16 * 4
    sub = (z > -709.7) & (z < -708.5)                     # 1 / (1 + e^-z) is subnormal: was NaN before the
    if sub.any():                                         # reciprocal scaled such quotients
        assert np.abs(h[sub] / ho[sub] - 1.0).max() < 1e-10
    # the fused predict kernel (exp + the same reciprocal on the DMMA path) on the same rows
    beta = rng.standard_normal((L, 2))
    model = rb.ElmModel(rb.ElmParams(d, L, 2, n + L), hid, beta)
    s, so = rb.predict(model, x), oracle.predict(hid.weights, hid.biases, beta, x)
    assert np.isfinite(s).all() and np.abs(s - so).max() <= 1e-11 * max(1.0, np.abs(so).max())


@pytest.mark.parametrize("n,d,L,m", [(7000, 24, 400, 60), (3001, 20, 130, 128), (20000, 40, 700, 100)])
def test_int8_accuracy_pass_vs_oracle(n, d, L, m):
    """K6i (oz_scores_kernel, m > 48): the training-accuracy pass from the Gram's digit planes gives the
    oracle's hit count (elm.cpp:278, 286-300) through the host-buffer train (two Gram parts, each with
    its own column exponents) and the device-resident train (one part); the ragged row counts leave
    partial 256-row tiles."""
    import oracle
    import torch

    x, t = rb.synth_classification(n, d, m, n + 7, m + 11)
    params = rb.ElmParams(d, L, m, L + 13)
    ref = oracle.train(d, L, m, L + 13, x, t, "rank", 0, 0.0)
    _, diag = rb.train(params, x, t, rb.SolverStrategy.rank_based())
    _, diag_d, _ = rb.train_device(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda(), params,
                                   rb.SolverStrategy.rank_based())
    print(f"n={n} L={L} m={m}: accuracy {diag.training_accuracy} / {diag_d.training_accuracy} "
          f"(oracle {ref['diag']['training_accuracy']})")
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]
    assert diag_d.training_accuracy == ref["diag"]["training_accuracy"]


def test_wide_inputs_fall_back_to_dmma_hidden_build():
    """d > 16384 exceeds the INT8 hidden build's int32 headroom (7 d 2^14 < 2^31): the DMMA hidden kernel
    builds H and its rows are scanned for the INT8 Gram's column exponents instead; the train still
    matches the oracle (pivots, rank, labels)."""
    import oracle

    n, d, L, m = 300, 16400, 40, 3
    x, t = rb.synth_classification(n, d, m, 91, 92)
    params = rb.ElmParams(d, L, m, 93)
    model, diag, order = rb.train(params, x, t, rb.SolverStrategy.rank_based(), return_order=True)
    ref = oracle.train(d, L, m, 93, x, t, "rank", 0, 0.0)
    assert diag.rank == ref["diag"]["rank"]
    assert order == ref["order"]
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]
    rel = np.linalg.norm(model.beta - ref["beta"]) / np.linalg.norm(ref["beta"])
    print(f"d={d}: beta rel {rel:.2e}")
    assert rel < 1e-6
