for c in c1 c4_250 c4_500 c4_1000 c4_2000 c4_4000 c4_8000 c5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
done
