"""One train() of an explicit shape (ncu captures of a chosen size): python tools/case_train.py N d L m [tol] [--predict]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_02436_b200 as rb  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n, d, L, m = (int(v) for v in args[:4])
tol = float(args[4]) if len(args) > 4 else 0.0
x, t = rb.synth_classification(n, d, m, 5, 6)
X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
beta, diag, hid = rb.train_device(X, T, rb.ElmParams(d, L, m, 7), rb.SolverStrategy.rank_based(tol))
if "--predict" in sys.argv:
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    rb.predict_device(X, W, B, beta, labels=labels)
torch.cuda.synchronize()
print("rank", diag.rank, "acc", diag.training_accuracy)
