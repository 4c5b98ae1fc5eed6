#!/bin/bash
# What the driver runs at round end, on the current HEAD: -m gpu suite (timed), smoke(), default bench, reference arm.
O=gpurun_out/head
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi > $O/smi.txt 2>&1
( time timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 ) > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
( time timeout 300 python __graft_entry__.py smoke ) > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
( time timeout 900 python bench.py ) > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
( time timeout 900 python bench.py --impl reference ) > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
echo done
