"""Measured C3 attention+remap layer timeline (one step after warm-up), same
per-step calls as bench.py, in the reference's Chrome-trace schema, plus a
per-rank summary (attention busy time, gaps, remap):
torchrun --nproc-per-node N tools/trace_layer.py OUT.json"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2509_21841_b200 import engine, trace, workloads as W  # noqa: E402
from paper_2509_21841_b200 import plan as P, remap as M, schedule as S  # noqa: E402
from paper_2509_21841_b200.program import build_rank_program  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
if world > 1:
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
ctx = engine.RankContext(rank, world, dev)
batch = W.c3_batch(world)
cluster = W.cluster_for(batch, world)
stager = engine.TableStager(dev)
hq, hkv, d = 32, 8, 128


def host_plan():
    plan = P.build_plan(batch, cluster)
    sched = S.build_schedule(plan)
    res = M.solve_remap(plan.tokens_per_rank, M.cost_matrix(cluster))
    prog = build_rank_program(plan, sched, rank, hq, res)
    return plan, sched, prog, engine.DeviceProgram(prog, dev, stager)


plan, sched, prog, devp = host_plan()
rows = prog.rows
q = torch.randn(rows, hq, d, device=dev, dtype=torch.bfloat16)
k = torch.randn(rows, hkv, d, device=dev, dtype=torch.bfloat16)
v = torch.randn(rows, hkv, d, device=dev, dtype=torch.bfloat16)
peer = engine.PeerBuffer(ctx, cluster.token_capacity, hq * d) if world > 1 else None
act = peer.buf if peer is not None else torch.empty(max(rows, prog.remap.linear_rows[rank]), hq * d, device=dev,
                                                     dtype=torch.bfloat16)
o = act[:rows].view(rows, hq, d)
lse = torch.empty(hq, max(rows, 1), device=dev)


def step():
    engine.attention_forward(plan, sched, q, k, v, ctx, prog, devp, out=(o, lse))
    if peer is not None:
        with ctx.span("compute", "remap.forward"):
            engine.remap_pull(prog.remap, peer, act, ctx)
        with ctx.span("compute", "remap.inverse"):
            engine.remap_pull(prog.remap, peer, act, ctx, inverse=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
ctx.tracer = trace.Tracer()
with ctx.span("compute", "layer.step"):
    step()
doc = trace.export(ctx.tracer, ctx, sys.argv[1])
if rank == 0:
    evs = doc["traceEvents"]
    for r in range(world):
        mine = sorted([e for e in evs if e["tid"].startswith(f"{r}.")], key=lambda e: e["ts"])
        st = [e for e in mine if e["name"] == "layer.step"][0]
        attn = [e for e in mine if e["name"].endswith(".attn")]
        busy = sum(e["dur"] for e in attn)
        gaps = sum(max(0.0, b["ts"] - (a["ts"] + a["dur"])) for a, b in zip(attn, attn[1:]))
        rem = sum(e["dur"] for e in mine if e["name"].startswith("remap"))
        first = attn[0]["ts"] - st["ts"] if attn else 0.0
        print(f"rank {r}: step {st['dur'] / 1e3:.2f} ms, attention {busy / 1e3:.2f} ms in {len(attn)} launches, "
              f"gaps between launches {gaps / 1e3:.2f} ms, first launch at +{first / 1e3:.2f} ms, remap {rem / 1e3:.2f} ms")
if world > 1:
    dist.destroy_process_group()
