#!/bin/bash
# Hidden-build epilogue experiment: stage-interleaved sigmoid batches (U = 2, 4, 8) vs the element-by-element form.
# Each variant library is swapped in; beta / pivot digests must be identical, hidden_kernel time is compared.
O=gpurun_out/hid_variants
mkdir -p $O
LIB=paper_2011_02436_b200/librbpelm_b200.so
cp $LIB /tmp/keep.so
for v in base u2 u4 u8; do
  cp tools/dbg/variants/$v.so $LIB
  python - "$v" >> $O/digests.txt 2>&1 <<'PY'
import hashlib, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2011_02436_b200 as rb
for (n, d, L, m) in [(2000, 16, 200, 2), (50000, 64, 1000, 10), (30000, 256, 1500, 100)]:
    x, t = rb.synth_classification(n, d, m, 1001, 2001)
    model, diag, order = rb.train(rb.ElmParams(d, L, m, 3001), x, t, rb.SolverStrategy.rank_based(), return_order=True)
    h = rb.hidden_matrix(model.hidden, x[:4000])
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
    print(sys.argv[1], (n, d, L, m), "rank", diag.rank, "H", dg(h), "beta", dg(model.beta), "order", dg(np.array(order)))
PY
  for c in c5 c4_8000 c2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>>$O/err.log | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', '$c', 'train %.3f ms'%d['train_ms'], 'hidden %.3f ms'%d['kernel_ms_per_step']['hidden_kernel'], 'clk', d['clocks']['sm_mhz'])
" >> $O/times.txt
  done
done
cp /tmp/keep.so $LIB
cat $O/digests.txt $O/times.txt
