#!/bin/bash
O=gpurun_out/pred
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_api_extras.py tests/test_ozaki_gpu.py tests/test_cpp_dropin.py -x -q -m gpu > $O/gpu.log 2>&1; echo "rc=$?" >> $O/gpu.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1
timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c2.log 2>&1
