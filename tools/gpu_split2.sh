#!/bin/bash
O=gpurun_out/split2
mkdir -p $O
export PYTHONUNBUFFERED=1
./tools/slice_check > $O/slice.log 2>&1; echo "rc=$?" >> $O/slice.log
./tools/ozaki_test check 5000 300 >> $O/slice.log 2>&1
./tools/ozaki_test time 500000 8292 2 >> $O/slice.log 2>&1
timeout 1200 python -m pytest tests/test_ozaki_gpu.py tests/test_gpu_parity.py -x -q -m gpu > $O/gpu.log 2>&1; echo "rc=$?" >> $O/gpu.log
for c in c1 c2 c4_250 c4_500 c4_1000 c4_8000 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
