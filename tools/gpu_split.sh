#!/bin/bash
O=gpurun_out/split
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -x -q -m gpu > $O/gpu.log 2>&1; echo "rc=$?" >> $O/gpu.log
for c in c1 c2 c4_250 c4_500 c4_1000 c4_2000; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
