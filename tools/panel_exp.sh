#!/bin/bash
O=gpurun_out/pexp
mkdir -p $O
for c in c4_4000 c4_8000 c4_2000; do
  for e in 0 1 2 3 0; do
    echo "EXP=$e" >> $O/log.txt
    RBPG_PANEL_EXP=$e timeout 300 python tools/panel_exp.py $c 5 >> $O/log.txt 2>&1
  done
done
