"""Train time and profiled panel / trailing time of one config (panel experiments)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n, d, L, m, _ = bench.CONFIGS[cfg]
x, t = rb.synth_classification(n, d, m, bench.SEED_X, bench.SEED_TEACHER)
X = torch.from_numpy(x).cuda()
T = torch.from_numpy(t).cuda()
p = rb.ElmParams(d, L, m, bench.SEED_W)
ctx = rb.context(0)
s = rb.SolverStrategy.rank_based()
for _ in range(3):
    beta, diag, _ = rb.train_device(X, T, p, s, ctx=ctx)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    beta, diag, _ = rb.train_device(X, T, p, s, ctx=ctx)
e1.record()
torch.cuda.synchronize()
train_ms = e0.elapsed_time(e1) / reps
ctx.set_profiling(True)
for _ in range(reps):
    rb.train_device(X, T, p, s, ctx=ctx)
torch.cuda.synchronize()
out = {k: round(ctx.profile(k)[0] / reps, 4) for k in ("panel_kernel", "syrk_trailing", "trsm_pair_kernel")}
ctx.set_profiling(False)
print(f"{cfg} rank {diag.rank} acc {diag.training_accuracy:.4f} train {train_ms:.4f} ms", out,
      f"beta[0,:3] {beta[0, :3].tolist()}")
