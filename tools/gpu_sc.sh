#!/bin/bash
O=gpurun_out/sc
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > $O/gpu.log 2>&1; echo "rc=$?" >> $O/gpu.log
for c in c2 c4_8000 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
