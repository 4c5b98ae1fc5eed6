#!/bin/bash
O=gpurun_out/hid
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_ozaki_gpu.py -x -q -s -m gpu > $O/oz.log 2>&1; echo "rc=$?" >> $O/oz.log
timeout 900 python -m pytest tests -x -q -m gpu > $O/gpu.log 2>&1; echo "rc=$?" >> $O/gpu.log
for c in c2 c4_8000 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
