#!/bin/bash
# Wide-panel evidence at C4 L=8000: per-phase cycle trace of the 32-wide panels, ncu of one wide panel launch.
O=gpurun_out/panel
mkdir -p $O
export PYTHONUNBUFFERED=1
RBPG_PANEL_TRACE=wide timeout 300 python tools/one_train.py c4_8000 1 > $O/trace_wide.log 2>&1
RBPG_PANEL_TRACE=1 timeout 300 python tools/one_train.py c4_4000 1 > $O/trace_c4_4000.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:panel_reg_kernel" -s 20 -c 1 -f -o $O/panel_wide \
    python tools/one_train.py c4_8000 1 > $O/panel_wide.log 2>&1
ncu -i $O/panel_wide.ncu-rep --page raw --csv > $O/panel_wide.csv 2>/dev/null
ncu -i $O/panel_wide.ncu-rep --page source --csv > $O/panel_wide_src.csv 2>/dev/null
echo done
