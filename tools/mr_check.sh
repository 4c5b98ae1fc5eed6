#!/bin/bash
# functional check of the N>1 bench path (2 gloo ranks sharing the one GPU; not a scaling number)
O=gpurun_out/mr
mkdir -p $O
export PYTHONUNBUFFERED=1
RBPG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 --config c4_1000 \
  --no-cpu-baseline > $O/gloo2_c4_1000.log 2>&1; echo "rc=$?" >> $O/gloo2_c4_1000.log
RBPG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 2 --warmup 3 --config c2 --scaling weak \
  --no-cpu-baseline > $O/gloo2_c2_weak.log 2>&1; echo "rc=$?" >> $O/gloo2_c2_weak.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 2 --warmup 3 --config c2 --no-cpu-baseline > $O/nccl1_c2.log 2>&1; echo "rc=$?" >> $O/nccl1_c2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --config c2 > $O/ref2_c2.log 2>&1; echo "rc=$?" >> $O/ref2_c2.log
