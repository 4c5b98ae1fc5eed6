"""Quick GPU-vs-oracle check used during development (run under gpurun)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check(n, d, L, m, seed=7, tol=0.0):
    x, t = rb.synth_classification(n, d, m, seed=11, teacher_seed=12)
    p = rb.ElmParams(d, L, m, seed)
    hid = rb.init_hidden(p)
    w, b = oracle.init_hidden(d, L, m, seed)
    assert np.array_equal(w, hid.weights) and np.array_equal(b, hid.biases)
    t0 = time.time()
    H = rb.hidden_matrix(hid, x)
    Ho = oracle.hidden_matrix(w, b, x)
    print(f"[{n}x{d} L={L}] H maxabs diff {np.abs(H - Ho).max():.3e}  ({time.time()-t0:.2f}s)")
    G = rb.gram(Ho)
    Go = oracle.gram(Ho)
    print("  gram rel", rel(G, Go), "sym", np.abs(G - G.T).max())
    f = rb.rank_revealing_factor(Ho, tol)
    oo, rk, tv, fo, mm = oracle.factor_gram(G, n, tol)
    print("  rank", f.permutation.rank, rk, "order equal", f.permutation.order == oo, "min margin", mm)
    if f.permutation.order != oo:
        diff = [i for i in range(L) if f.permutation.order[i] != oo[i]]
        print("  first order diffs", diff[:10], [f.permutation.order[i] for i in diff[:5]], [oo[i] for i in diff[:5]])
    print("  factor rel", rel(f.factor, fo))
    model, diag = rb.train(p, x, t, rb.SolverStrategy.rank_based(tol))
    ref = oracle.train(d, L, m, seed, x, t, "rank", 0, tol)
    print("  beta rel", rel(model.beta, ref["beta"]), "rank", diag.rank, ref["diag"]["rank"], "acc",
          diag.training_accuracy, ref["diag"]["training_accuracy"], "hidden_s", diag.hidden_seconds, "solve_s",
          diag.solve_seconds)
    sc = rb.predict(model, x)
    so = oracle.predict(ref["w"], ref["b"], ref["beta"], x)
    print("  labels equal", bool((sc.argmax(1) == so.argmax(1)).all()), "score rel", rel(sc, so))


if __name__ == "__main__":
    oracle.set_threads(16)
    check(2000, 16, 200, 2)
    check(3000, 20, 300, 3)
    check(50000, 64, 1000, 10)
