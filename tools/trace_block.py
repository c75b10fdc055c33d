"""Measured C5 block timeline (one step after warm-up) in the reference's
Chrome-trace schema: torchrun --nproc-per-node N tools/trace_block.py OUT.json"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2509_21841_b200 import block as B, engine, trace, workloads as W  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
if world > 1:
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
ctx = engine.RankContext(rank, world, dev)
batch = W.c4_batch()
blk = B.ZeppelinBlock(W.cluster_for(batch, world), B.BlockWeights.random(dev), ctx)
blk.prepare(batch)
x = torch.randn(blk.rows[1], B.HIDDEN, device=dev, dtype=torch.bfloat16)
for _ in range(2):
    blk.forward(x)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
ctx.tracer = trace.Tracer()
blk.forward(x)
doc = trace.export(ctx.tracer, ctx, sys.argv[1])
if rank == 0:
    print(len(doc["traceEvents"]), "events ->", sys.argv[1])
if world > 1:
    dist.destroy_process_group()
