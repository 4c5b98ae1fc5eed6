"""Row-sharded multi-rank path on the device: two ranks (gloo, both on cuda:0) run the product's
orchestration (sharded.train_sharded with DeviceStages: sm_100a augmented Gram per shard ->
all-reduce -> replicated device solve -> all-reduced hit count) and are checked against the
oracle on the concatenated rows: identical pivots and rank, bitwise-identical beta on both ranks,
beta within the oracle's 1-vs-2-shard reduction-order floor, equal training accuracy.

Two ranks sharing one GPU only exercise the orchestration and the host-staged all-reduce; the
product's NCCL path is the same code with backend "nccl" on one GPU per rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, n, d, L, m, out):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2011_02436_b200 as rb
    from paper_2011_02436_b200 import sharded

    x, t = rb.synth_classification(n * world, d, m, seed=41, teacher_seed=42)
    row0, rows = sharded.shard_rows(n * world, world, rank)
    xl = torch.from_numpy(np.ascontiguousarray(x[row0:row0 + rows])).cuda()
    tl = torch.from_numpy(np.ascontiguousarray(t[row0:row0 + rows])).cuda()
    params = rb.ElmParams(d, L, m, 43)
    beta, diag, _, order = sharded.train_sharded(xl, tl, params, rb.SolverStrategy.rank_based(), n * world,
                                                 stages=sharded.DeviceStages(rb.context(0)))
    out[rank] = (beta.cpu().numpy(), diag.rank, [int(v) for v in order], diag.training_accuracy)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,d,L,m", [(3000, 16, 200, 2), (6000, 32, 400, 5)])
def test_sharded_device_world2_matches_oracle(n, d, L, m):
    import oracle
    import paper_2011_02436_b200 as rb

    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), n, d, L, m, out), nprocs=world, join=True)
        res = dict(out)
    x, t = rb.synth_classification(n * world, d, m, seed=41, teacher_seed=42)
    ref = oracle.train(d, L, m, 43, x, t, "rank")
    b0, r0, o0, a0 = res[0]
    b1, r1, o1, a1 = res[1]
    assert np.array_equal(b0, b1), "ranks disagree on beta"
    assert r0 == r1 == ref["diag"]["rank"] == L
    assert o0 == o1 == ref["order"], "pivot order differs from the oracle"
    rel = np.linalg.norm(b0 - ref["beta"]) / np.linalg.norm(ref["beta"])
    assert rel <= 1e-9, rel
    assert a0 == a1 == ref["diag"]["training_accuracy"]


@pytest.mark.parametrize("L,m", [(400, 5), (201, 2)])
def test_device_stage_odd_leading_dimension(L, m):
    """Stage API into caller buffers whose leading dimension is odd (L + m odd): the Gram kernels'
    16-byte stores go through an aligned staging buffer; results equal the even-ld call."""
    import paper_2011_02436_b200 as rb

    n, d = 4000, 16
    x, t = rb.synth_classification(n, d, m, seed=51, teacher_seed=52)
    p = rb.ElmParams(d, L, m, 53)
    hid = rb.init_hidden(p)
    X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    M = L + m
    g_odd = torch.empty((M, M), dtype=torch.float64, device="cuda")
    g_even = torch.empty((M, M + 1), dtype=torch.float64, device="cuda")[:, :M]
    rb.gram_stage_device_aug(X, T, W, B, g_odd)
    rb.gram_stage_device_aug(X, T, W, B, g_even)
    assert torch.equal(g_odd, g_even)
    rb.gram_stage_device_aug(X, T, W, B, g_odd, accumulate=True)
    assert torch.equal(g_odd, 2 * g_even)
    h = torch.sigmoid(X @ W + B)
    gh = torch.empty((L, L), dtype=torch.float64, device="cuda")
    rb.gram_device(h, gh)
    assert torch.allclose(gh, g_even[:L, :L], rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("fixed_order", [False, True])
def test_train_multi_native_entry(fixed_order):
    """rbpg_train_multi (single-process multi-device C entry) on the one GPU here: upload of the shard,
    augmented Gram, packed-triangle exchange (NCCL path taken only with > 1 device), replicated solve.
    With one device its Gram is the device-resident train()'s, so beta is bitwise equal."""
    import paper_2011_02436_b200 as rb

    n, d, L, m = 20000, 32, 700, 6
    x, t = rb.synth_classification(n, d, m, 81, 82)
    params = rb.ElmParams(d, L, m, 83)
    model, diag, order = rb.train_multi(params, x, t, rb.SolverStrategy.rank_based(), devices=[0],
                                        fixed_order=fixed_order, return_order=True)
    X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    beta_d, diag_d, _, order_d = rb.train_device(X, T, params, rb.SolverStrategy.rank_based(), return_order=True)
    assert order == order_d and diag.rank == diag_d.rank == L
    assert np.array_equal(model.beta, beta_d.cpu().numpy())
    assert diag.training_accuracy == diag_d.training_accuracy
    with pytest.raises(ValueError, match="one context per device"):
        rb.train_multi(params, x, t, rb.SolverStrategy.rank_based(), devices=[0, 0])
