"""Functional check of the sharded stages under torch.distributed (any backend, any rank count
on the visible GPUs): per-rank Gram checksum before / after the all-reduce and the solve."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2011_02436_b200 as rb  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count())
torch.cuda.set_device(dev)
dist.init_process_group(os.environ.get("RBPG_DIST_BACKEND", "nccl"))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, L, m, _ = bench.CONFIGS[cfg]
xh, th = rb.synth_classification(n, d, m, bench.SEED_X, bench.SEED_TEACHER, row0=rank * n)
X, T = torch.from_numpy(xh).to(dev), torch.from_numpy(th).to(dev)
p = rb.ElmParams(d, L, m, bench.SEED_W)
hid = rb.init_hidden(p)
W = torch.from_numpy(hid.weights).to(dev)
B = torch.from_numpy(hid.biases.reshape(-1)).to(dev)
ctx = rb.context(dev.index)
G = torch.empty((L + m, L + m), dtype=torch.float64, device=dev)
rb.gram_stage_device_aug(X, T, W, B, G, ctx=ctx)
torch.cuda.synchronize()
print(f"rank {rank}: local G trace {G.diagonal().sum().item():.6e} sum {G.sum().item():.6e}", flush=True)
dist.all_reduce(G)
torch.cuda.synchronize()
print(f"rank {rank}: reduced G trace {G.diagonal().sum().item():.6e} sum {G.sum().item():.6e}", flush=True)
beta, diag = rb.solve_stage_device_aug(G, L, m, n * world, rb.SolverStrategy.rank_based(), ctx=ctx)
print(f"rank {rank}: rank {diag.rank} beta sum {beta.sum().item():.12e}", flush=True)
hits = rb.accuracy_stage_device(X, T, W, B, beta, ctx=ctx)
print(f"rank {rank}: local hits {hits} of {n}", flush=True)
dist.destroy_process_group()
