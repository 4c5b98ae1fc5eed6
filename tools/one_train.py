"""One device-resident train() of a BASELINE config (for ncu / compute-sanitizer captures).

  python tools/one_train.py <config> [reps] [--predict]

--predict also runs one fused batched predict (K6b) over the training rows after the train."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = args[0] if args else "c2"
reps = int(args[1]) if len(args) > 1 else 1
n, d, L, m, _ = bench.CONFIGS[cfg]
x, t = rb.synth_classification(n, d, m, bench.SEED_X, bench.SEED_TEACHER)
X = torch.from_numpy(x).cuda()
T = torch.from_numpy(t).cuda()
p = rb.ElmParams(d, L, m, bench.SEED_W)
for _ in range(reps):
    beta, diag, hid = rb.train_device(X, T, p, rb.SolverStrategy.rank_based())
if "--predict" in sys.argv:
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    rb.predict_device(X, W, B, beta, labels=labels)
torch.cuda.synchronize()
print("rank", diag.rank, "acc", diag.training_accuracy)
