#!/bin/bash
# Round-2 evidence of the INT8-Gram state on one B200: bench sweep, launch lists (C5 default bench,
# C2), ncu --set full of the INT8 Gram (C4 L=8000, C5), the slice/colmax passes and the C2 panel.
O=gpurun_out/prof2
mkdir -p $O
export PYTHONUNBUFFERED=1
for c in c1 c2 c4_250 c4_500 c4_1000 c4_2000 c4_4000 c4_8000; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/sweep.jsonl 2>> $O/sweep.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c5.log 2>&1; echo "rc=$?" >> $O/ncu_launch_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c2.csv \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1; echo "rc=$?" >> $O/ncu_launch_c2.log
cap() {  # name regex skip config [extra]
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -f -o $O/$1 \
    python tools/one_train.py $4 1 $5 > $O/$1.log 2>&1
  echo "rc=$?" >> $O/$1.log
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.csv 2>/dev/null
}
cap ozgram_c4_8000 "oz_gram2_kernel" 0 c4_8000
cap ozslice_c5 "oz_slice_kernel" 0 c5
cap ozcolmax_c5 "oz_colmax_kernel" 0 c5
cap ozgram_c2 "oz_gram2_kernel" 0 c2
cap ozgram_c5 "oz_gram2_kernel" 0 c5
echo profile-done
