#!/bin/bash
# K1i epilogue with the in-range sigmoid: digests vs the previous library, hidden_kernel times, H tests.
O=gpurun_out/hid_fast
mkdir -p $O
LIB=paper_2011_02436_b200/librbpelm_b200.so
cp $LIB /tmp/new.so
for v in base new; do
  if [ $v = base ]; then cp tools/dbg/variants/base.so $LIB; else cp /tmp/new.so $LIB; fi
  python - "$v" >> $O/digests.txt 2>&1 <<'PY'
import hashlib, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2011_02436_b200 as rb
for (n, d, L, m) in [(2000, 16, 200, 2), (50000, 64, 1000, 10), (30000, 256, 1500, 100), (1003, 20, 77, 3)]:
    x, t = rb.synth_classification(n, d, m, 1001, 2001)
    model, diag, order = rb.train(rb.ElmParams(d, L, m, 3001), x, t, rb.SolverStrategy.rank_based(), return_order=True)
    h = rb.hidden_matrix(model.hidden, x[:4099])
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
    print(sys.argv[1], (n, d, L, m), "rank", diag.rank, "H", dg(h), "beta", dg(model.beta), "order", dg(np.array(order)))
PY
  for c in c2 c4_1000 c4_8000 c5; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>>$O/err.log | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', '$c', 'train %.3f ms'%d['train_ms'], 'hidden %.3f ms'%d['kernel_ms_per_step']['hidden_kernel'], 'clk', d['clocks']['sm_mhz'])
" >> $O/times.txt
  done
done
cp /tmp/new.so $LIB
timeout 900 python -m pytest tests/test_ozaki_gpu.py -q -s -k "hidden" > $O/pytest_hidden.log 2>&1; echo "rc=$?" >> $O/pytest_hidden.log
cat $O/digests.txt $O/times.txt; tail -5 $O/pytest_hidden.log
