#!/bin/bash
O=gpurun_out/hid2
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_ozaki_gpu.py -x -q -m gpu > $O/oz.log 2>&1; echo "rc=$?" >> $O/oz.log
for c in c2 c4_8000 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_hidden -c 1 -f -o $O/hid_c4_8000 \
  python tools/one_train.py c4_8000 1 > $O/ncu.log 2>&1
ncu -i $O/hid_c4_8000.ncu-rep --page raw --csv > $O/hid_c4_8000.csv 2>/dev/null
ncu -i $O/hid_c4_8000.ncu-rep --page source --csv > $O/hid_c4_8000_src.csv 2>/dev/null
ncu -i $O/hid_c4_8000.ncu-rep --page details --csv > $O/hid_c4_8000_det.csv 2>/dev/null
