#!/bin/bash
# Trailing-update evidence at C4 L=8000: device timeline of every panel / trailing launch, ncu --set full
# of one wide-phase (rank-32) and one narrow-phase (rank-64) trail_kernel launch.
O=gpurun_out/trail
mkdir -p $O
export PYTHONUNBUFFERED=1
RBPG_DEVICE_TIMELINE=1 timeout 300 python tools/one_train.py c4_8000 2 > $O/timeline.log 2>&1; echo "rc=$?" >> $O/timeline.log
cap() {  # name regex skip config
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -f -o $O/$1 \
    python tools/one_train.py $4 1 > $O/$1.log 2>&1
  echo "rc=$?" >> $O/$1.log
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page source --csv > $O/$1_src.csv 2>/dev/null
}
cap trail_wide "trail_kernel" 10 c4_8000
cap trail_narrow "trail_kernel" 140 c4_8000
cap ozhidden_c4 "oz_hidden_kernel" 0 c4_8000
echo done
