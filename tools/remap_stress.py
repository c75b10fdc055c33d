"""Remap stress layouts S1/S2 alone (bench.run_remap_stress), one JSON line."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_21841_b200 import engine  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
ctx = engine.RankContext(rank, world, dev)
res = bench.run_remap_stress(ctx, dev, world, rank, None)
if rank == 0:
    for name, r in res.items():
        print(name, {k: ((round(v["GB_per_s_busiest_sender"], 1), round(v["ms"], 4)) if isinstance(v, dict) else v)
                     for k, v in r.items() if k in ("nccl_all_to_allv", "fused_peer_store", "fused_peer_load", "copy_engine_pull", "copy_engine_push", "handshake_only", "all_paths_equal")})
dist.destroy_process_group()
