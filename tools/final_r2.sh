#!/bin/bash
# Round-2 final evidence on one B200: default bench (C5) + reference arm, sweep, parity numbers,
# launch list of the default bench, ncu --set full of the INT8 kernels at C5.
O=gpurun_out/final
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
for c in c1 c2 c4_250 c4_500 c4_1000 c4_2000 c4_4000 c4_8000; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/sweep.jsonl 2>> $O/sweep.err
done
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > $O/bench_c2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -m gpu > $O/parity_s.log 2>&1; echo "rc=$?" >> $O/parity_s.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c5.log 2>&1; echo "rc=$?" >> $O/ncu_launch_c5.log
cap() {  # name regex skip config
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -f -o $O/$1 \
    python tools/one_train.py $4 1 > $O/$1.log 2>&1
  echo "rc=$?" >> $O/$1.log
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.csv 2>/dev/null
}
cap ozhidden_c5 "oz_hidden_kernel" 0 c5
cap ozscores_c5 "oz_scores_kernel" 0 c5
cap ozslice_c5 "oz_slice_kernel" 0 c5
cap ozgram_c5 "oz_gram2_kernel" 0 c5
rm -f $O/*.ncu-rep
echo done
