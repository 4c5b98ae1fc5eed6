"""Device SVD pseudo-inverse (pinv_svd, linalg.cpp:68-87) and the solve_direct branch that uses it
(elm.cpp:108-122: N < L, or a singular Gram after the rank path / SingularSplit fallbacks).

The SVD itself is an implementation choice in both the reference (Eigen BDCSVD) and the oracle
(scalar one-sided Jacobi); where singular values sit near the cut rel * s_max the pseudo-inverse
is ill-determined and two correct SVDs disagree.  So every comparison is gated on the
SVD-implementation floor: the distance between the oracle and numpy's LAPACK SVD on the same
input (gate max(1e-9, 4 * floor)).  The reference's own pinv tests (Penrose conditions, known
answers) run in test_reference_suite.py on both implementations.
"""
import numpy as np
import pytest

import oracle
import paper_2011_02436_b200 as rb
from impls import pinv, rel_fro

pytestmark = pytest.mark.gpu


def sig_features(n, d, L, seed=5):
    x, _ = rb.synth_classification(n, d, 2, seed, seed + 1)
    w, b = oracle.init_hidden(d, L, 2, seed + 2)
    return oracle.hidden_matrix(w, b, x)


@pytest.mark.parametrize("shape", [(300, 40), (40, 300), (1000, 200), (200, 1000), (777, 133)])
def test_pinv_svd_vs_oracle_and_lapack(shape):
    h = sig_features(shape[0], 8, shape[1])
    got = rb.pinv_svd(h)
    want = oracle.pinv_svd(h)
    floor = rel_fro(pinv(h), want)
    err = rel_fro(got, want)
    print(f"{shape}: pinv rel {err:.2e} (oracle-vs-LAPACK floor {floor:.2e})")
    assert err <= max(1e-9, 4 * floor)


def test_pinv_svd_exact_rank_deficiency_and_zero_columns():
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, (400, 9)) @ rng.uniform(-1, 1, (9, 70))
    a[:, 13] = 0.0
    a[:, 40] = a[:, 2]
    got = rb.pinv_svd(a)
    assert rel_fro(got, pinv(a)) < 1e-9
    assert np.abs(got[13]).max() == 0.0  # a zero column has a zero row in the pseudo-inverse
    assert rel_fro(a @ got @ a, a) < 1e-12


def test_solve_direct_wide_min_norm():
    """direct strategy with N < L: beta = pinv(H) Y is the minimum-norm interpolant."""
    x, t = rb.synth_classification(150, 6, 3, 31, 32)
    params = rb.ElmParams(6, 300, 3, 33)
    model, diag = rb.train(params, x, t, rb.SolverStrategy.direct())
    ref = oracle.train(6, 300, 3, 33, x, t, "direct", 0, 0.0)
    assert diag.used_svd_path and ref["diag"]["used_svd_path"]
    h = oracle.hidden_matrix(ref["w"], ref["b"], x)
    floor = rel_fro(h @ (pinv(h) @ t), h @ ref["beta"])
    err = rel_fro(h @ model.beta, h @ ref["beta"])
    print(f"wide direct: fitted rel {err:.2e} (floor {floor:.2e}), beta rel {rel_fro(model.beta, ref['beta']):.2e}")
    assert err <= max(1e-9, 4 * floor)
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]


def test_svd_fallback_branch_degenerate():
    """d = 2 inputs, L = 640: H is numerically rank ~40 with singular values straddling the cut.  The
    rank path finds r < L, the Schur block stays singular after the ridge retry (SingularSplit) and
    solve_direct falls back to pinv_svd (elm.cpp:216-225, 119-121)."""
    x, t = rb.synth_classification(700, 2, 2, 700, 3)
    model, diag, order = rb.train(rb.ElmParams(2, 640, 2, 642), x, t, rb.SolverStrategy.rank_based(),
                                  return_order=True)
    ref = oracle.train(2, 640, 2, 642, x, t, "rank", 0, 0.0)
    assert diag.fallback_to_direct and diag.used_svd_path
    assert ref["diag"]["fallback_to_direct"] and ref["diag"]["used_svd_path"]
    h = oracle.hidden_matrix(ref["w"], ref["b"], x)
    # rank attribution: the oracle factorisation of the GPU's own Gram (the train path's, i.e. the INT8
    # digit-plane Gram of [H T]) reproduces the GPU rank
    import torch

    G = torch.empty((640, 640), dtype=torch.float64, device="cuda")
    HtT = torch.empty((640, 2), dtype=torch.float64, device="cuda")
    rb.gram_stage_device(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda(),
                         torch.from_numpy(model.hidden.weights).cuda(),
                         torch.from_numpy(model.hidden.biases.reshape(-1)).cuda(), G, HtT, keep_h=False)
    o2, r2, _, _, margin = oracle.factor_gram(G.cpu().numpy(), 700, 0.0)
    # singular values straddle the cut here by construction: the stop test at the boundary pivot is
    # decided by the factorisations' own rounding (FMA / blocked dot products on the device, sequential
    # sums in the oracle), so the two ranks may differ by one; the branch taken must not
    assert abs(diag.rank - r2) <= 1
    first = next((i for i, (a, b) in enumerate(zip(order, o2)) if a != b), None)
    print(f"rank gpu {diag.rank} / oracle {ref['diag']['rank']} / oracle-on-GPU-Gram {r2}; "
          f"pivot orders first differ at {first} (min pivot margin {margin:.1e})")
    floor = rel_fro(h @ (pinv(h) @ t), h @ ref["beta"])
    err = rel_fro(h @ model.beta, h @ ref["beta"])
    print(f"fitted rel {err:.2e} (SVD floor {floor:.2e})")
    assert err <= max(1e-9, 4 * floor)
    assert diag.training_accuracy == ref["diag"]["training_accuracy"]
