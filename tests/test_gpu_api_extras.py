"""Device tests of the drop-in pieces added in round 2: the fused batched predict (K6b), the block
split solve, SpdFactor with a device-resident factor, matmul / matmul_at on the DMMA GEMM, the packed
exchange helpers of the row-sharded path, and the kept-H invalidation of the stage API."""
import numpy as np
import pytest

import oracle
import paper_2011_02436_b200 as rb

pytestmark = pytest.mark.gpu


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n,d,L,m", [(1000, 16, 200, 2), (777, 64, 1000, 10), (5000, 24, 333, 33),
                                     (300, 256, 520, 100), (129, 3, 31, 1), (4100, 40, 257, 65)])
def test_predict_fused_vs_oracle(n, d, L, m):
    """rbpg_predict (host buffers) and rbpg_predict_device run the fused sigma(XW+b) beta kernel; scores
    match the oracle's predict to rounding, labels exactly (elm.cpp:282-300)."""
    import torch

    x, t = rb.synth_classification(n, d, m, n + 1, d + 2)
    hid = rb.init_hidden(rb.ElmParams(d, L, m, L + 3))
    rng = np.random.default_rng(L)
    beta = rng.standard_normal((L, m))
    model = rb.ElmModel(rb.ElmParams(d, L, m, 0), hid, beta)
    s = rb.predict(model, x)
    so = oracle.predict(hid.weights, hid.biases, beta, x)
    assert rel_fro(s, so) < 1e-12
    assert (s.argmax(1) == so.argmax(1)).all()
    X = torch.from_numpy(x).cuda()
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    Bt = torch.from_numpy(beta).cuda()
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    scores = torch.empty((n, m), dtype=torch.float64, device="cuda")
    rb.predict_device(X, W, B, Bt, scores=scores, labels=labels)
    assert np.array_equal(scores.cpu().numpy(), s)  # same kernel, same bits
    assert (labels.cpu().numpy() == so.argmax(1)).all()


def test_predict_label_ties_lowest_index():
    """Exact ties between classes go to the lowest index (elm.cpp:291-296): beta with two identical
    columns makes every row tie between them."""
    n, d, L = 500, 8, 40
    x, _ = rb.synth_classification(n, d, 2, 5, 6)
    hid = rb.init_hidden(rb.ElmParams(d, L, 3, 7))
    beta = np.random.default_rng(1).standard_normal((L, 3))
    beta[:, 2] = beta[:, 1]
    beta[:, 0] -= 100.0
    s = rb.predict(rb.ElmModel(rb.ElmParams(d, L, 3, 0), hid, beta), x)
    assert np.array_equal(s[:, 1], s[:, 2])
    assert (s.argmax(1) == 1).all()


def test_accuracy_stage_does_not_reuse_stale_h():
    """a kept H must only serve the exact inputs that built it.  train_device keeps [H T]
    for its own X; an accuracy pass on a different X of the same shape recomputes (fused kernel)."""
    import torch

    n, d, L, m = 4000, 20, 300, 4
    x, t = rb.synth_classification(n, d, m, 11, 12)
    x2, t2 = rb.synth_classification(n, d, m, 13, 14)
    params = rb.ElmParams(d, L, m, 15)
    X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    beta, diag, hid = rb.train_device(X, T, params, rb.SolverStrategy.rank_based())
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    X2, T2 = torch.from_numpy(x2).cuda(), torch.from_numpy(t2).cuda()
    hits2 = rb.accuracy_stage_device(X2, T2, W, B, beta)
    so = oracle.predict(hid.weights, hid.biases, beta.cpu().numpy(), x2)
    assert hits2 == int((so.argmax(1) == t2.argmax(1)).sum())
    hits1 = rb.accuracy_stage_device(X, T, W, B, beta)
    assert hits1 / n == diag.training_accuracy


@pytest.mark.parametrize("n,c1,c2,m", [(400, 30, 50, 3), (2000, 128, 200, 7), (3000, 300, 1, 2)])
def test_solve_block_split_vs_oracle(n, c1, c2, m):
    """elm.cpp:124-156 through rbpg_solve_block_split."""
    rng = np.random.default_rng(n + c1)
    h = rng.uniform(0, 1, (n, c1 + c2))
    y = np.eye(m)[rng.integers(0, m, n)]
    b1, b2 = rb.solve_block_split(h[:, :c1], h[:, c1:], y)
    o1, o2, od = oracle.solve_block_split(h[:, :c1], h[:, c1:], y)
    fit, fit_o = h @ np.vstack([b1, b2]), h @ np.vstack([o1, o2])
    assert rel_fro(fit, fit_o) < 1e-9
    assert not od["ridge_applied"]


def test_solve_block_split_errors_and_ridge():
    rng = np.random.default_rng(9)
    h = rng.uniform(0, 1, (200, 10))
    y = np.eye(2)[rng.integers(0, 2, 200)]
    with pytest.raises(rb.ShapeError, match="row counts differ"):
        rb.solve_block_split(h[:100, :4], h[:, 4:], y)
    with pytest.raises(rb.ShapeError, match="at least as many samples"):
        rb.solve_block_split(h[:5, :4], h[:5, 4:], y[:5])
    # duplicated column across the split: D is singular, the ridge rescues it (test_elm.cpp:120-136)
    hd = np.hstack([h[:, :5], h[:, :1]])
    diag = rb.SolveDiagnostics()
    b1, b2 = rb.solve_block_split(hd[:, :5], hd[:, 5:], y, 1e-8, diag)
    o1, o2, od = oracle.solve_block_split(hd[:, :5], hd[:, 5:], y)
    assert diag.ridge_applied == bool(od["ridge_applied"])
    assert rel_fro(hd @ np.vstack([b1, b2]), hd @ np.vstack([o1, o2])) < 1e-7


def test_spd_factor_device_resident():
    rng = np.random.default_rng(4)
    a = rng.standard_normal((300, 200))
    m = a.T @ a + np.eye(200)
    f = rb.SpdFactor(m)
    assert f.dim() == 200
    for k in (1, 5, 70):
        rhs = rng.standard_normal((200, k))
        assert rel_fro(f.solve(rhs), np.linalg.solve(m, rhs)) < 1e-12
    with pytest.raises(rb.ShapeError):
        f.solve(np.ones((3, 1)))
    with pytest.raises(rb.SingularMatrix) as e:
        rb.SpdFactor(np.diag([4.0, 0.0, 1.0]))
    assert e.value.pivot_index == 1


@pytest.mark.parametrize("ar,ac,bc", [(1, 1, 1), (70, 33, 9), (513, 129, 65), (64, 64, 64)])
def test_matmul_dmma(ar, ac, bc):
    """matrix.cpp:69-87 on the device (reference pin test_matrix.cpp:42-47: 1e-13 vs a triple loop)."""
    rng = np.random.default_rng(ar + ac)
    a = rng.standard_normal((ar, ac))
    b = rng.standard_normal((ac, bc))
    assert np.abs(rb.matmul(a, b) - oracle.matmul(a, b)).max() < 1e-13 * max(1.0, np.abs(a).sum(1).max() * np.abs(b).max())
    b2 = rng.standard_normal((ar, bc))
    assert np.allclose(rb.matmul_at(a, b2), a.T @ b2, rtol=1e-13, atol=1e-12)
    with pytest.raises(rb.ShapeError):
        rb.matmul(a, np.ones((ac + 1, 2)))
    with pytest.raises(rb.ShapeError):
        rb.matmul_at(a, np.ones((ar + 1, 2)))


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1010, 4197])
def test_pack_unpack_and_fixed_order_sum_device(n):
    import torch

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    sym = a + a.T
    g = torch.from_numpy(sym).cuda()
    packed = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device="cuda")
    rb.pack_lower_device(g, packed)
    ref = sym[np.tril_indices(n)]  # row-major lower triangle: (i, j <= i) at i(i+1)/2 + j
    assert np.array_equal(packed.cpu().numpy(), ref)
    out = torch.full((n, n), np.nan, dtype=torch.float64, device="cuda")
    rb.unpack_lower_device(packed, out)
    assert np.array_equal(out.cpu().numpy(), sym)
    parts = torch.from_numpy(rng.standard_normal((5, 1000))).cuda()
    s = torch.empty(1000, dtype=torch.float64, device="cuda")
    rb.sum_parts_device(parts, s)
    p = parts.cpu().numpy()
    assert np.array_equal(s.cpu().numpy(), (((p[0] + p[1]) + p[2]) + p[3]) + p[4])


def test_two_contexts_same_device():
    """Kernel attributes are tracked per (device, kernel): a second context reuses them."""
    c1, c2 = rb.Context(0), rb.Context(0)
    x, t = rb.synth_classification(3000, 16, 2, 1, 2)
    p = rb.ElmParams(16, 1100, 2, 3)  # > 48 KB shared-memory kernels (panel, TRSM cluster)
    m1, d1 = rb.train(p, x, t, rb.SolverStrategy.rank_based(), ctx=c1)
    m2, d2 = rb.train(p, x, t, rb.SolverStrategy.rank_based(), ctx=c2)
    assert np.array_equal(m1.beta, m2.beta)
    c1.close()
    c2.close()
