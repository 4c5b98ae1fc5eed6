#!/bin/bash
# Wide-panel G prefetch: digests + panel / trailing times at C4 L=8000, per-phase trace, C5 bench.
O=gpurun_out/pf
mkdir -p $O
export PYTHONUNBUFFERED=1
for c in c4_8000 c4_8000; do
  timeout 300 python tools/panel_exp.py $c 5 >> $O/digests.txt 2>&1
done
RBPG_PANEL_TRACE=wide timeout 300 python tools/one_train.py c4_8000 1 > $O/trace_wide.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1
timeout 300 python bench.py --config c4_8000 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4_8000.log 2>&1
echo done
