for v in 0 65 66; do for c in c4_8000 c5 c2; do RBPG_TRAIL_VARIANT=$v timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>>gpurun_out/r7.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('v=$v', '$c', round(d['ms_per_step'],2), {k:round(x,2) for k,x in d['kernel_ms_per_step'].items()})" >> gpurun_out/r7_trail.txt; done; done
RBPG_TRAIL_VARIANT=65 timeout 900 python -m pytest tests -q -m gpu -x -k "c4_sweep and (2000 or 8000) or c5_standin or ragged or C2" >> gpurun_out/r7_trail.txt 2>&1
