"""One train() of an explicit shape for compute-sanitizer: python tools/sanitize_case.py N d L m [tol]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_02436_b200 as rb  # noqa: E402

n, d, L, m = (int(v) for v in sys.argv[1:5])
tol = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
x, t = rb.synth_classification(n, d, m, 5, 6)
X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
beta, diag, _ = rb.train_device(X, T, rb.ElmParams(d, L, m, 7), rb.SolverStrategy.rank_based(tol))
torch.cuda.synchronize()
print("rank", diag.rank, "acc", diag.training_accuracy)
