#!/bin/bash
# fused predict kernel (K6b) with the in-range sigmoid: predict times before / after, predict parity tests
O=gpurun_out/pred_fast
mkdir -p $O
LIB=paper_2011_02436_b200/librbpelm_b200.so
cp $LIB /tmp/new.so
for v in base new; do
  if [ $v = base ]; then cp tools/dbg/variants/base.so $LIB; else cp /tmp/new.so $LIB; fi
  for c in c1 c2 c4_1000 c4_4000; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>>$O/err.log | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['predict']; print('$v', '$c', 'predict rows', p['rows'], '%.4f ms'%p['ms'], '%.2f TF/s'%p['TFLOP/s'], 'frac %.3f'%p['frac_fp64_peak'], 'train %.3f ms'%d['train_ms'])
" >> $O/times.txt
  done
done
cp /tmp/new.so $LIB
timeout 900 python -m pytest tests -q -m gpu -k "predict or saturating or baseline_configs or api_extras or golden" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cat $O/times.txt; tail -4 $O/pytest.log
