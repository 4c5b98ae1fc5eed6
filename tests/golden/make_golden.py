"""Regenerate tests/golden/c1_oracle.json: the oracle's outputs on the C1 workload
(seeded synthetic inputs; see bench.py CONFIGS).  Run: python tests/golden/make_golden.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

SEED_X, SEED_T, SEED_W = 1001, 2001, 3001
x, t = rb.synth_classification(2000, 16, 2, SEED_X, SEED_T)
r = oracle.train(16, 200, 2, SEED_W, x, t, "rank")
out = {"config": "C1: N=2000 d=16 L=200 m=2, rank strategy, default tol", "seed_x": SEED_X, "seed_teacher": SEED_T,
       "seed_w": SEED_W, "rank": r["diag"]["rank"], "order": r["order"],
       "training_accuracy": r["diag"]["training_accuracy"], "min_pivot_margin": r["diag"]["min_pivot_margin"],
       "beta": r["beta"].tolist()}
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c1_oracle.json"), "w"))
print("wrote c1_oracle.json", out["rank"], out["training_accuracy"])
