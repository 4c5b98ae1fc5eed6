"""One device-resident train() of a BASELINE config (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n, d, L, m = bench.CONFIGS[cfg]
x, t = rb.synth_classification(n, d, m, bench.SEED_X, bench.SEED_TEACHER)
X = torch.from_numpy(x).cuda()
T = torch.from_numpy(t).cuda()
p = rb.ElmParams(d, L, m, bench.SEED_W)
for _ in range(reps):
    beta, diag, _ = rb.train_device(X, T, p, rb.SolverStrategy.rank_based())
torch.cuda.synchronize()
print("rank", diag.rank, "acc", diag.training_accuracy)
