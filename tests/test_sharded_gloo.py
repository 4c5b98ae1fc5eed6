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


class OracleStages:
    def __init__(self, tol=0.0):
        self.tol = tol

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


def _worker(rank, world, port, n, d, L, m, out):
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
                                         rb.SolverStrategy.rank_based(), n, stages=OracleStages())
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
