"""Panel-variant experiment: train time, panel/trailing time and bitwise equality of order and beta
against the default variant (run once per RBPG_PANEL_EXP value)."""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n, d, L, m, _ = bench.CONFIGS[cfg]
x, t = rb.synth_classification(n, d, m, bench.SEED_X, bench.SEED_TEACHER)
X = torch.from_numpy(x).cuda()
T = torch.from_numpy(t).cuda()
p = rb.ElmParams(d, L, m, bench.SEED_W)
ctx = rb.context(0)
s = rb.SolverStrategy.rank_based()
for _ in range(2):
    beta, diag, _, order = rb.train_device(X, T, p, s, ctx=ctx, return_order=True)
torch.cuda.synchronize()
ctx.set_profiling(True)
for _ in range(reps):
    rb.train_device(X, T, p, s, ctx=ctx)
torch.cuda.synchronize()
pm = ctx.profile("panel_kernel")[0] / reps
tm = ctx.profile("syrk_trailing")[0] / reps
ctx.set_profiling(False)
h = hashlib.sha256(beta.cpu().numpy().tobytes() + np.array(order, dtype=np.int64).tobytes()).hexdigest()[:16]
print(f"{cfg} panels {pm:.2f} ms trailing {tm:.2f} ms rank {diag.rank} digest {h}")
