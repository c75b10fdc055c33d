"""Run the C2 attention launch (64K github seed-0 batch, all local) a few
times; used as the ncu target (python tools/attn_c2.py [iters])."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_21841_b200 import ops, plan as P, schedule as S, workloads as W  # noqa: E402
from paper_2509_21841_b200.engine import DeviceProgram  # noqa: E402
from paper_2509_21841_b200.program import build_rank_program  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
batch = W.c2_batch("github", 0)
plan = P.build_plan(batch, W.cluster_for(batch, 1))
prog = build_rank_program(plan, S.build_schedule(plan), 0, 32)
dev = torch.device("cuda", 0)
dp = DeviceProgram(prog, dev)
t = prog.rows
q = torch.randn(t, 32, 128, device=dev, dtype=torch.bfloat16)
k = torch.randn(t, 8, 128, device=dev, dtype=torch.bfloat16)
v = torch.randn(t, 8, 128, device=dev, dtype=torch.bfloat16)
o = torch.empty_like(q)
lse = torch.empty(32, t, device=dev)
for _ in range(iters):
    ops.attn_fwd(q, k, v, dp.local.items, dp.local.n, dp.local.segs, o, lse)
torch.cuda.synchronize()
print("pairs", prog.pairs_per_head(), "items", dp.local.n)
