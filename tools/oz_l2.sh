#!/bin/bash
# L2-reuse experiment for the INT8 Gram: item k-length (OZ_KPER k-steps) x launch-order block (OZ_PBLOCK)
O=gpurun_out/ozl2
mkdir -p $O
for kper in 512 256 128; do
  for pb in 3 6 12; do
    echo "kper=$kper pblock=$pb" >> $O/time.log
    OZ_KPER=$kper OZ_PBLOCK=$pb timeout 120 ./tools/ozaki_test time 100000 8010 3 >> $O/time.log 2>&1
  done
done
for pb in 3 6 12; do
  echo "C5 kper=512 pblock=$pb" >> $O/time.log
  OZ_PBLOCK=$pb timeout 200 ./tools/ozaki_test time 500000 8292 2 >> $O/time.log 2>&1
done
echo "C5 kper=256 pblock=6" >> $O/time.log
OZ_KPER=256 OZ_PBLOCK=6 timeout 200 ./tools/ozaki_test time 500000 8292 2 >> $O/time.log 2>&1
for v in "512 3" "128 3" "128 12"; do
  set -- $v
  OZ_KPER=$1 OZ_PBLOCK=$2 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    -k regex:oz_gram2 -c 1 ./tools/ozaki_test time 100000 8010 1 > $O/ncu_k$1_b$2.log 2>&1
done
echo done
