"""Row-sharded multi-rank path on CPU: world_size 2 over gloo.

Runs the product's orchestration (paper_2011_02436_b200.sharded.train_sharded:
shard -> local Gram -> all-reduce -> replicated solve -> all-reduced hit count)
with test-only CPU stages built from the oracle, and checks that every rank gets
a bitwise-identical beta and the same pivots/rank as the unsharded oracle, with
beta inside the oracle's reduction-order floor."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pack_lower_np(g):
    """Host statement of the packed layout the device kernels use: (i, j <= i) at i(i+1)/2 + j."""
    n = g.shape[0]
    return np.concatenate([g[i, :i + 1] for i in range(n)])


def unpack_lower_np(p, n):
    g = np.zeros((n, n))
    for i in range(n):
        g[i, :i + 1] = p[i * (i + 1) // 2:(i + 1) * (i + 2) // 2]
    return np.tril(g) + np.tril(g, -1).T


class OracleStages:
    def __init__(self, tol=0.0):
        self.tol = tol

    def pack(self, g):
        return torch.from_numpy(pack_lower_np(g.numpy()))

    def unpack(self, packed, g):
        g.copy_(torch.from_numpy(unpack_lower_np(packed.numpy(), g.shape[0])))

    def sum_parts(self, parts, out):
        acc = parts[0].clone()
        for r in range(1, parts.shape[0]):
            acc = acc + parts[r]  # rank order, one rounded add per element
        out.copy_(acc)

    def as_tensor(self, x, like):
        return torch.as_tensor(np.asarray(x, dtype=np.float64))

    def gram_aug(self, x, t, w, b):
        import oracle

        h = oracle.hidden_matrix(w.numpy(), b.numpy().reshape(1, -1), x.numpy())
        self._h = h
        return torch.from_numpy(oracle.gram(np.hstack([h, t.numpy()])))

    def solve_aug(self, gaug, L, m, n_total, strategy):
        import oracle
        import paper_2011_02436_b200 as rb

        g = np.ascontiguousarray(gaug.numpy()[:L, :L])
        htt = torch.from_numpy(np.ascontiguousarray(gaug.numpy()[:L, L:L + m]))
        order, rank, _, f, _ = oracle.factor_gram(g, n_total, strategy.rank_tol)
        assert rank == g.shape[0]
        x = oracle.solve_factored_gram(f, order, rank, htt.numpy()[order])
        beta = np.empty_like(x)
        beta[order] = x
        d = rb.SolveDiagnostics(strategy=strategy.describe(), rank=rank, rank_known=True)
        return torch.from_numpy(beta), d, order

    def hits(self, x, t, w, b, beta):
        s = self._h @ beta.numpy()
        return int((s.argmax(1) == t.numpy().argmax(1)).sum())


def _worker(rank, world, port, n, d, L, m, out, fixed_order=False):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2011_02436_b200 as rb
    from paper_2011_02436_b200.sharded import shard_rows, train_sharded

    oracle.set_threads(1)
    row0, nl = shard_rows(n, world, rank)
    x, t = rb.synth_classification(nl, d, m, 1001, 2001, row0=row0)
    params = rb.ElmParams(d, L, m, 3001)
    beta, diag, _, order = train_sharded(torch.from_numpy(x), torch.from_numpy(t), params,
                                         rb.SolverStrategy.rank_based(), n, stages=OracleStages(),
                                         fixed_order=fixed_order)
    out[rank] = (beta.numpy().copy(), list(order), diag.training_accuracy)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_train_matches_unsharded(world):
    import oracle
    import paper_2011_02436_b200 as rb

    n, d, L, m = 2001, 16, 200, 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, d, L, m, out), nprocs=world, join=True)
    b0, o0, acc0 = out[0]
    for r in range(1, world):
        br, orr, accr = out[r]
        assert np.array_equal(b0, br) and o0 == orr and acc0 == accr  # replicated solve: bitwise identical
    x, t = rb.synth_classification(n, d, m, 1001, 2001)
    ref = oracle.train(d, L, m, 3001, x, t, "rank")
    assert o0 == ref["order"]
    assert np.linalg.norm(b0 - ref["beta"]) / np.linalg.norm(ref["beta"]) < 1e-9
    assert acc0 == ref["diag"]["training_accuracy"]


def test_packed_layout_roundtrip():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((37, 37))
    g = a + a.T
    p = pack_lower_np(g)
    assert p.size == 37 * 38 // 2
    assert np.array_equal(unpack_lower_np(p, 37), g)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fixed_order_equals_oracle_shard_sum(world):
    """fixed_order=True: all-gather of the packed partials + a rank-order sum.  The Gram every rank
    factors is then bitwise the oracle's world-shard Gram (gram_sharded sums contiguous row shards
    in shard order), so beta and pivots are bitwise those of the oracle run on that Gram."""
    import oracle
    import paper_2011_02436_b200 as rb

    n, d, L, m = 2001, 16, 200, 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, d, L, m, out, True), nprocs=world, join=True)
    x, t = rb.synth_classification(n, d, m, 1001, 2001)
    w, b = oracle.init_hidden(d, L, m, 3001)
    h = oracle.hidden_matrix(w, b, x)
    gaug = oracle.gram(np.hstack([h, t]), world)
    order, rank, _, f, _ = oracle.factor_gram(np.ascontiguousarray(gaug[:L, :L]), n)
    xs = oracle.solve_factored_gram(f, order, rank, gaug[:L, L:L + m][order])
    beta = np.empty_like(xs)
    beta[order] = xs
    for r in range(world):
        br, orr, _ = out[r]
        assert orr == order
        assert np.array_equal(br, beta)
