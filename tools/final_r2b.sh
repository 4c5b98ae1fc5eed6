#!/bin/bash
# refresh after the K1i epilogue change: launch list of the default bench, ncu --set full of oz_hidden_kernel at C5
O=gpurun_out/final_b
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c5.log 2>&1; echo "rc=$?" >> $O/ncu_launch_c5.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:oz_hidden_kernel" -s 0 -c 1 -f -o $O/ozhidden_c5 \
  python tools/one_train.py c5 1 > $O/ozhidden_c5.log 2>&1; echo "rc=$?" >> $O/ozhidden_c5.log
ncu -i $O/ozhidden_c5.ncu-rep --page raw --csv > $O/ozhidden_c5.csv 2>/dev/null
rm -f $O/*.ncu-rep
echo done
