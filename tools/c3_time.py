"""BASELINE C3 (rank-deficient: N=20000, d=32 = 16 base + 16 linear combinations, L=2000 with 500
exact duplicate nodes, m=5) on the device: augmented Gram stage with the duplicated hidden layer,
then the rank-based solve at tol 1e-6 (rank 1500, Schur block path with the ridge retry), timed
with CUDA events on the launching stream (inputs resident, L2 flushed between steps)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_02436_b200 as rb  # noqa: E402

n, base, L, m = 20000, 16, 2000, 5
x, t = rb.synth_rank_deficient(n, base, m, 1002, 4001, 2002)
hid0 = rb.init_hidden(rb.ElmParams(2 * base, L, m, 3002))
hid, _, _ = rb.duplicate_nodes(hid0, 500, 5001)
X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
W = torch.from_numpy(hid.weights).cuda()
B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
G = torch.empty((L + m, L + m), dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
strat = rb.SolverStrategy.rank_based(1e-6)


def step():
    rb.gram_stage_device_aug(X, T, W, B, G)
    return rb.solve_stage_device_aug(G, L, m, n, strat)


for _ in range(3):
    beta, diag = step()
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    beta, diag = step()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"C3 rank {diag.rank} ridge_applied {diag.ridge_applied} fallback {diag.fallback_to_direct} "
      f"train (Gram stage + solve) median {statistics.median(ts):.3f} ms")
