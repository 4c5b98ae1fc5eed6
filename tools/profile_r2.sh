#!/bin/bash
# Round-2 evidence run on one B200 (gpurun): multi-rank bench functional check, launch list of the
# default bench, ncu --set full captures of the top kernels, compute-sanitizer on the cluster kernels.
O=gpurun_out/prof
mkdir -p $O
export PYTHONUNBUFFERED=1
# 1. bench under torchrun: 2 ranks on the one GPU with gloo (functional check of the N>1 path)
RBPG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --config c4_1000 \
  --no-cpu-baseline > $O/bench_gloo2.log 2>&1; echo "rc=$?" >> $O/bench_gloo2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --config c2 > $O/ref_torchrun2.log 2>&1
echo "rc=$?" >> $O/ref_torchrun2.log
# 2. launch list of the default bench command (C5 shard)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
# 3. full-set captures
cap() {  # name regex skip config [extra]
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -f -o $O/$1 \
    python tools/one_train.py $4 1 $5 > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.csv 2>/dev/null
}
cap gram_c5 "syrk_kernel" 0 c5
cap gramdiag_c5 "syrk_diag_kernel" 0 c5
cap trail_c4_8000 "trail_kernel" 2 c4_8000
cap panelgrid_c4_8000 "panel_kernel_t" 4 c4_8000
cap hidden_c1 "hidden_kernel" 0 c1
cap hidden_c5 "hidden_kernel" 0 c5
cap scores_c2 "scores_kernel" 0 c2
cap predict_c5 "predict_kernel" 0 c5 --predict
cap panel_c2 "panel_reg_kernel" 3 c2
# 4. compute-sanitizer on the cluster / st.async kernels (small shapes)
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/case_train.py 3000 16 600 3 > $O/sanitize_${tool}_reg.log 2>&1
  echo "rc=$?" >> $O/sanitize_${tool}_reg.log
  timeout 1200 compute-sanitizer --tool $tool python tools/case_train.py 5000 8 4300 2 > $O/sanitize_${tool}_grid.log 2>&1
  echo "rc=$?" >> $O/sanitize_${tool}_grid.log
done
echo profile-done
