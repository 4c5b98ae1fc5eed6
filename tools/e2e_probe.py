"""Where the end-to-end train() time goes at a BASELINE config: raw pinned H2D rate, device-resident
train, and the C-ABI train from host buffers (RBPG_HOST_TRACE prints the host-side split)."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, L, m, _ = bench.CONFIGS[cfg]
xh, th = rb.synth_classification(n, d, m, bench.SEED_X, bench.SEED_TEACHER)
xp = torch.from_numpy(xh).pin_memory()
tp = torch.from_numpy(th).pin_memory()
dx = torch.empty_like(xp, device="cuda")
dt = torch.empty_like(tp, device="cuda")
for _ in range(3):
    dx.copy_(xp, non_blocking=True)
    dt.copy_(tp, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dx.copy_(xp, non_blocking=True)
    dt.copy_(tp, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
nb = xp.numel() * 8 + tp.numel() * 8
print(f"H2D {nb / 1e6:.1f} MB: {statistics.median(ts):.3f} ms ({nb / statistics.median(ts) / 1e6:.1f} GB/s)")
p = rb.ElmParams(d, L, m, bench.SEED_W)
strat = rb.SolverStrategy.rank_based()
ctx = rb.context(0)
for _ in range(3):
    rb.train(p, xp.numpy(), tp.numpy(), strat, ctx=ctx)
te = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rb.train(p, xp.numpy(), tp.numpy(), strat, ctx=ctx)
    te.append(time.perf_counter() - t0)
print(f"e2e train: median {statistics.median(te) * 1e3:.3f} ms min {min(te) * 1e3:.3f} ms")
X, T = dx, dt
for _ in range(3):
    rb.train_device(X, T, p, strat, ctx=ctx)
td = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rb.train_device(X, T, p, strat, ctx=ctx)
    torch.cuda.synchronize()
    td.append(time.perf_counter() - t0)
print(f"device-resident train (wall): median {statistics.median(td) * 1e3:.3f} ms")
