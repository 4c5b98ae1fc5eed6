#!/bin/bash
# INT8 Gram weight split A/B: group 1 from weight 6 (current) vs from weight 5
O=gpurun_out/ozsplit
mkdir -p $O
for w in 5 6; do
  echo "== W0G1=$w" >> $O/log.txt
  ./tools/ozaki_test_w$w check 5000 300 >> $O/log.txt 2>&1
  ./tools/ozaki_test_w$w check 40000 200 >> $O/log.txt 2>&1
done
for rep in 1 2; do
  for w in 5 6; do
    echo "== W0G1=$w rep $rep" >> $O/log.txt
    timeout 300 ./tools/ozaki_test_w$w time 500000 8292 3 >> $O/log.txt 2>&1
    timeout 300 ./tools/ozaki_test_w$w time 100000 8010 3 >> $O/log.txt 2>&1
    timeout 300 ./tools/ozaki_test_w$w time 50000 1010 5 >> $O/log.txt 2>&1
  done
done
