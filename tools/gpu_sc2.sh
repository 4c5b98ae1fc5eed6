#!/bin/bash
O=gpurun_out/sc2
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_ozaki_gpu.py -x -q -s -m gpu > $O/oz.log 2>&1; echo "rc=$?" >> $O/oz.log
for c in c2 c4_8000 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
