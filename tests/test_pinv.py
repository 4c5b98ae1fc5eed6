"""Rank-path pseudo-inverse H^+ (SURVEY §8 a11): P (F F^T)^-1 P^T H^T for full-rank H.

Oracle definition: the full-rank solve of elm.cpp:202-214 with right-hand side H^T (oracle
`oracle_pseudo_inverse`, solve_factored_gram per column).  Independent check: numpy's SVD
pseudo-inverse (the reference's pinv_svd, linalg.cpp:68-87, is the same mathematical object for
full-rank H).  Bars: order and rank bit-exact; H^+ within relative Frobenius max(1e-9, 4 * floor),
the floor being the oracle-vs-SVD difference (both are backward-stable; their gap measures the
conditioning).  Sizes beyond the oracle: H^+ T must reproduce the rank-path beta of solve_beta.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2011_02436_b200 as rb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def hidden(n, d, L, seed=5):
    x, _ = rb.synth_classification(n, d, 2, seed, seed + 1)
    w, b = oracle.init_hidden(d, L, 2, seed + 2)
    return oracle.hidden_matrix(w, b, x)


# ---------------------------------------------------------------------------- CPU (oracle)
def test_oracle_pinv_matches_svd_pinv():
    h = hidden(600, 12, 80)
    p, order, rank = oracle.pseudo_inverse(h)
    assert rank == 80 and sorted(order) == list(range(80))
    assert rel_fro(p, np.linalg.pinv(h)) < 1e-8
    assert np.allclose(p @ h, np.eye(80), atol=1e-6)


def test_oracle_pinv_rank_deficient_raises_like_solve_factored_gram():
    h = hidden(400, 8, 30)
    h[:, 7] = h[:, 3]
    with pytest.raises(oracle.OracleFailure) as e:
        oracle.pseudo_inverse(h)
    assert e.value.code == 2 and "rank-deficient (29 of 30)" in str(e.value)


class OracleStages:
    def gram_of(self, h):
        return torch.from_numpy(oracle.gram(h.numpy()))

    def pinv_block(self, g, h, n_total, tol):
        order, rank, _, f, _ = oracle.factor_gram(g.numpy(), n_total, tol)
        x = oracle.solve_factored_gram(f, order, rank, np.ascontiguousarray(h.numpy().T[order]))
        out = np.empty_like(x)
        out[order] = x
        return torch.from_numpy(out), order, rank


def _worker(rank, world, port, n, d, L, out):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2011_02436_b200.sharded import pseudo_inverse_sharded, shard_rows

    oracle.set_threads(1)
    row0, nl = shard_rows(n, world, rank)
    h = hidden(n, d, L)[row0:row0 + nl]
    blk, order, rk = pseudo_inverse_sharded(torch.from_numpy(np.ascontiguousarray(h)), n, stages=OracleStages())
    out[rank] = (row0, blk.numpy().copy(), list(order), rk)
    dist.destroy_process_group()


def test_sharded_pinv_gloo_world2():
    n, d, L = 900, 10, 60
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, port, n, d, L, out), nprocs=2, join=True)
    full, order, rank = oracle.pseudo_inverse(hidden(n, d, L))
    got = np.concatenate([out[r][1] for r in range(2)], axis=1)
    assert out[0][2] == out[1][2] == order and out[0][3] == rank == L
    assert rel_fro(got, full) < 1e-9


# ---------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(2000, 16, 200), (3000, 24, 257), (6000, 32, 500), (1500, 40, 1)])
def test_pinv_parity_vs_oracle(shape):
    n, d, L = shape
    h = hidden(n, d, L)
    want, order_o, rank_o = oracle.pseudo_inverse(h)
    got, order, rank = rb.pseudo_inverse(h)
    assert rank == rank_o == L and order == order_o
    floor = rel_fro(want, np.linalg.pinv(h))
    err = rel_fro(got, want)
    print(f"{shape}: H+ rel {err:.3e} (oracle-vs-SVD floor {floor:.3e})")
    assert err <= max(1e-9, 4 * floor)


@pytest.mark.gpu
def test_pinv_rank_deficient_raises():
    # an exact duplicate column: after its twin is pivoted, its running diagonal is a rounding residual
    # of order eps * d (sign included), so below ~sqrt(eps) whether it falls under the cut is decided
    # by rounding -- in the reference as here.  Engineered dependencies are therefore tested at the
    # reference tests' own tolerance, 1e-6 (test_linalg.cpp:92-116, test_elm.cpp:138-151).
    h = hidden(2000, 16, 200)
    h[:, 50] = h[:, 10]
    with pytest.raises(ValueError, match=r"rank-deficient \(199 of 200\)"):
        rb.pseudo_inverse(h, 1e-6)


@pytest.mark.gpu
def test_pinv_c2_reproduces_rank_path_beta():
    """C2 (50000 x 1000): H^+ T equals solve_beta's rank-path beta (same factorisation, same pivots)."""
    x, t = rb.synth_classification(50000, 64, 10, 1001, 2001)
    hl = rb.init_hidden(rb.ElmParams(64, 1000, 10, 3001))
    h = rb.hidden_matrix(hl, x)
    p, order, rank = rb.pseudo_inverse(h)
    assert rank == 1000 and p.shape == (1000, 50000)
    d = rb.SolveDiagnostics()
    beta = rb.solve_beta(h, t, rb.SolverStrategy.rank_based(), d)
    err = rel_fro(p @ t, beta)
    print(f"C2: |H+ T - beta| / |beta| = {err:.3e}")
    assert err < 1e-8
    # left-inverse property on a column sample
    idx = np.arange(0, 1000, 37)
    assert np.abs(p[idx] @ h - np.eye(1000)[idx]).max() < 1e-6


@pytest.mark.gpu
def test_pinv_stage_device_column_blocks():
    """Row shards on one device: the per-shard column blocks from the accumulated Gram tile H^+."""
    n, d, L = 5000, 20, 300
    h = hidden(n, d, L)
    want, order_o, _ = oracle.pseudo_inverse(h)
    dev = torch.device("cuda:0")
    g = torch.zeros((L, L), dtype=torch.float64, device=dev)
    bounds = [(0, 1700), (1700, 3301), (3301, 5000)]
    shards = [torch.from_numpy(np.ascontiguousarray(h[a:b])).to(dev) for a, b in bounds]
    for i, hs in enumerate(shards):
        rb.gram_device(hs, g, accumulate=i > 0)
    blocks = []
    for hs in shards:
        blk, order, rank = rb.pseudo_inverse_stage_device(g, hs, n)
        assert order == order_o and rank == L
        blocks.append(blk.cpu().numpy())
    got = np.concatenate(blocks, axis=1)
    assert rel_fro(got, want) <= max(1e-9, 4 * rel_fro(want, np.linalg.pinv(h)))
