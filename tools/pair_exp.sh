#!/bin/bash
# Gram item pairing change: bitwise digests (beta + pivot order) vs the previous pairing, Gram times, C5 bench.
O=gpurun_out/pair
mkdir -p $O
export PYTHONUNBUFFERED=1
for c in c2 c4_4000 c4_8000; do
  timeout 300 python tools/panel_exp.py $c 5 >> $O/digests.txt 2>&1
done
for c in c2 c4_1000 c4_8000; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/sweep.jsonl 2>> $O/sweep.err
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1
timeout 900 python -m pytest tests/test_ozaki_gpu.py tests/test_gpu_parity.py -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
echo done
