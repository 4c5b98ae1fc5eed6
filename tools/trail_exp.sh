#!/bin/bash
O=gpurun_out/texp2
mkdir -p $O
for c in c4_8000 c4_4000 c4_8000 c4_4000; do
  timeout 300 python tools/panel_exp.py $c 5 >> $O/log.txt 2>&1
done
