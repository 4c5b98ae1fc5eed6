#!/bin/bash
# Quick HEAD check on one B200: GPU suite (timed), smoke, default bench, C2 and C4 L=8000 lines.
O=gpurun_out/head
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi > $O/smi.txt 2>&1
( time timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 ) > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
for c in c2 c4_8000; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/sweep.jsonl 2>> $O/sweep.err
done
echo done
