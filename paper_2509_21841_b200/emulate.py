"""Run every rank of a plan in ONE process on ONE GPU.

Used to validate the multi-GPU execution with the real sm_100a kernels when
only one B200 is available.  The forward runs the PRODUCTION executor
(``engine.attention_steps``): each emulated rank has its own context, compute
stream and comm stream, and its ring KV buffers / epoch flags in a
``RingTransport`` whose peer addresses are plain device pointers instead of
CUDA-IPC mappings — the hops are the same ``zp_ring_hop`` copy-engine pulls
and stream flag waits.

The members' step generators are interleaved ring step by ring step with a
device synchronisation between steps.  Every flag a step waits for is written
by an earlier step, so no flag wait ever blocks here.  This matters only in
one process: a flag edge is invisible to CUDA's scheduler, which may
serialise two streams of one process in either order (measured: the g=8
config-3 plan deadlocks with 8 hardware queues and completes with 32).  In a
real job every flag edge crosses processes, and each process's own work is
ordered by CUDA-visible stream / event edges only.
"""

from __future__ import annotations

import math

import torch

from . import ops
from .engine import DeviceProgram, RankContext, RingTransport, attention_steps, ring_rows_needed
from .program import build_rank_program


def gather_rank(seq_tensors: dict, plan, rank: int, device) -> torch.Tensor:
    parts = [seq_tensors[f.sequence_id][f.start:f.end] for f in plan.fragments[rank]]
    return torch.cat(parts, 0).to(device).contiguous()


def emulate_ranks_on_one_gpu(plan, sched, sq: dict, sk: dict, sv: dict, device="cuda", parity: bool = False,
                             softmax_scale: float | None = None):
    """Every rank's attention_forward on one GPU.  Returns [(o, lse)] per rank
    in attention layout (o bf16; fp32 with ``parity``: V converted to fp16 and
    the parity kernel, zp_attn_fwd_parity)."""
    hq = next(iter(sq.values())).shape[1]
    hkv, d = next(iter(sk.values())).shape[1:]
    ad = ops.HeadAdapter(hq, hkv, d)
    if not ad.identity:  # e.g. config 1's 4 heads x d64 (MHA): padded / head-duplicated layout
        adapted = {s: ad.inputs(sq[s], sk[s], sv[s]) for s in sq}
        outs = emulate_ranks_on_one_gpu(plan, sched, {s: a[0] for s, a in adapted.items()},
                                        {s: a[1] for s, a in adapted.items()}, {s: a[2] for s, a in adapted.items()},
                                        device, parity, softmax_scale=d ** -0.5)
        return [ad.outputs(o, lse) for o, lse in outs]
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else softmax_scale
    dev = torch.device(device)
    world = plan.num_ranks
    ctxs = [RankContext(r, world, dev) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    rows = ring_rows_needed(sched)
    if rows:
        for c, t in zip(ctxs, RingTransport.local_group(ctxs, rows, 2 * hkv * d * 2)):
            c.ring = t
    progs = [build_rank_program(plan, sched, r, hq) for r in range(world)]
    devs = [DeviceProgram(p, dev) for p in progs]
    q = [gather_rank(sq, plan, r, dev) for r in range(world)]
    k = [gather_rank(sk, plan, r, dev) for r in range(world)]
    v = [gather_rank(sv, plan, r, dev) for r in range(world)]
    if parity:
        v = [x.to(torch.float16) for x in v]
    outs = [(torch.zeros(q[r].shape, dtype=torch.float32 if parity else torch.bfloat16, device=dev),
             torch.full((hq, max(p.rows, 1)), float("-inf"), device=dev)) for r, p in enumerate(progs)]
    torch.cuda.synchronize(dev)  # tables, inputs and outputs are ready before the rank streams start
    gens = [attention_steps(plan, sched, q[r], k[r], v[r], ctxs[r], progs[r], devs[r], outs[r][0], outs[r][1],
                            scale) for r in range(world)]

    def advance(r):
        with torch.cuda.stream(streams[r]):
            return next(gens[r], None)

    for ri, rs in enumerate(sched.rings()):
        for step in range(rs.ring.group_size + 1):
            for m in rs.ring.members:
                tag = advance(m)
                if tag != (ri, step):
                    raise AssertionError(f"rank {m}: expected ring step {(ri, step)}, got {tag}")
            torch.cuda.synchronize(dev)  # every flag the next step waits for is written
    for r in range(world):
        while advance(r) is not None:
            pass
    torch.cuda.synchronize(dev)
    return outs


def emulate_backward_on_one_gpu(plan, sched, sq: dict, sk: dict, sv: dict, sdo: dict, outs, device="cuda"):
    """Every rank's attention_backward on one GPU through the production
    executor (``engine.attention_backward_steps``): LocalTask gradients, ring
    rounds with the KV sets pulled hop by hop and the dK/dV running totals
    pulled, added and forwarded by the same copy-engine / flag protocol, the
    own set's total returned after the last round.  ``outs`` are the
    forward's (o, lse) per rank.  Returns [(dq, dk, dv) fp32] per rank in
    attention layout."""
    from .engine import BwdDeviceProgram, attention_backward_steps
    from .program import build_bwd_program
    hq = next(iter(sq.values())).shape[1]
    hkv, d = next(iter(sk.values())).shape[1:]
    scale = 1.0 / math.sqrt(d)
    dev = torch.device(device)
    world = plan.num_ranks
    ctxs = [RankContext(r, world, dev) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    rows = ring_rows_needed(sched)
    if rows:
        ts = RingTransport.local_group(ctxs, rows, 2 * hkv * d * 2)
        RingTransport.attach_grad_local(ts, rows, hkv * d)
        for c, t in zip(ctxs, ts):
            c.ring = t
    progs = [build_rank_program(plan, sched, r, hq) for r in range(world)]
    devs = [DeviceProgram(p, dev) for p in progs]
    bdevs = [BwdDeviceProgram(build_bwd_program(p, hkv), dev) for p in progs]
    q = [gather_rank(sq, plan, r, dev) for r in range(world)]
    k = [gather_rank(sk, plan, r, dev) for r in range(world)]
    v = [gather_rank(sv, plan, r, dev) for r in range(world)]
    do = [gather_rank(sdo, plan, r, dev) for r in range(world)]
    grads, deltas = [], []
    for r in range(world):
        o, lse = outs[r]
        delta = torch.empty_like(lse)
        if progs[r].rows:
            ops.attn_bwd_prep(o, do[r], delta)
        deltas.append(delta)
        grads.append(tuple(torch.zeros(x.shape, dtype=torch.float32, device=dev) for x in (q[r], k[r], k[r])))
    torch.cuda.synchronize(dev)
    gens = [attention_backward_steps(plan, sched, q[r], k[r], v[r], do[r], outs[r][1], deltas[r], *grads[r],
                                     ctxs[r], progs[r], bdevs[r], devs[r], scale) for r in range(world)]

    def advance(r):
        with torch.cuda.stream(streams[r]):
            return next(gens[r], None)

    for ri, rs in enumerate(sched.rings()):
        for step in range(rs.ring.group_size + 2):
            for m in rs.ring.members:
                tag = advance(m)
                if tag != (ri, step):
                    raise AssertionError(f"rank {m}: expected ring step {(ri, step)}, got {tag}")
            torch.cuda.synchronize(dev)  # every flag the next step waits for is written
    for r in range(world):
        while advance(r) is not None:
            pass
    torch.cuda.synchronize(dev)
    return grads


def emulate_remap_on_one_gpu(layout, xs: list, method: str = "pull", inverse: bool = False, device="cuda"):
    """The fused remap kernels (zp_remap_pull / zp_remap_push with their
    ready/done epoch handshakes) for every rank of ``layout`` on one GPU.
    ``xs[r]``: rank r's rows ([A_r, ...] forward, [B_r, ...] inverse).  Each
    rank runs on its own stream; the three stages are enqueued stage by stage
    across ranks (every rank's ready before any move), so a spinning ready
    kernel never sits in front of the peer stage it waits for.  Returns each
    rank's output rows (linear layout forward, attention layout inverse)."""
    from .engine import PeerBuffer, pull_tables, push_tables, remap_pull, remap_push
    dev = torch.device(device)
    world = layout.world
    ctxs = [RankContext(r, world, dev) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    row_elems = xs[0][0].numel() if xs[0].shape[0] else xs[1][0].numel()
    cap = max(max(layout.attn_rows), max(layout.linear_rows), 1)
    bufs = PeerBuffer.local_group(ctxs, cap, row_elems, xs[0].dtype)
    rows_in = layout.linear_rows if inverse else layout.attn_rows
    rows_out = layout.attn_rows if inverse else layout.linear_rows
    for r in range(world):
        bufs[r].buf[:rows_in[r]].copy_(xs[r].reshape(rows_in[r], row_elems))
    if method == "pull":
        tabs = [pull_tables(layout, r, inverse, dev) for r in range(world)]
    else:
        tabs = [push_tables(layout, r, inverse, dev) for r in range(world)]
    torch.cuda.synchronize(dev)
    for phase in (1, 2, 4):
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                if method == "pull":
                    remap_pull(layout, bufs[r], bufs[r].buf, ctxs[r], inverse=inverse, tables=tabs[r], phases=phase)
                else:
                    remap_push(layout, bufs[r].buf[:rows_in[r]], bufs[r], ctxs[r], inverse=inverse,
                               tables=tabs[r], phases=phase)
    torch.cuda.synchronize(dev)
    return [bufs[r].buf[:rows_out[r]].clone() for r in range(world)]
