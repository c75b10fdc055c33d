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
    """Backward of ``emulate_ranks_on_one_gpu``: every rank's LocalTask and
    ring-round gradients with ``zp_attn_bwd``; a ring's partial dK/dV travel
    with its KV set (device copies instead of NCCL) and return to the owner
    after the last round.  ``outs`` are the forward's (o, lse) per rank.
    Returns [(dq, dk, dv) fp32] per rank in attention layout."""
    from .program import build_bwd_program
    from .engine import BwdDeviceProgram
    hq = next(iter(sq.values())).shape[1]
    hkv, d = next(iter(sk.values())).shape[1:]
    scale = 1.0 / math.sqrt(d)
    dev = torch.device(device)
    progs = [build_rank_program(plan, sched, r, hq) for r in range(plan.num_ranks)]
    devs = [DeviceProgram(p, dev) for p in progs]
    bdevs = [BwdDeviceProgram(build_bwd_program(p, hkv), dev) for p in progs]
    q = [gather_rank(sq, plan, r, device) for r in range(plan.num_ranks)]
    k = [gather_rank(sk, plan, r, device) for r in range(plan.num_ranks)]
    v = [gather_rank(sv, plan, r, device) for r in range(plan.num_ranks)]
    do = [gather_rank(sdo, plan, r, device) for r in range(plan.num_ranks)]
    grads, deltas = [], []
    for r, bd in enumerate(bdevs):
        o, lse = outs[r]
        delta = torch.empty_like(lse)
        if progs[r].rows:
            ops.attn_bwd_prep(o, do[r], delta)
        dq = torch.zeros(q[r].shape, dtype=torch.float32, device=dev)
        dk = torch.zeros(k[r].shape, dtype=torch.float32, device=dev)
        dv = torch.zeros(k[r].shape, dtype=torch.float32, device=dev)
        if bd.local.n:
            ops.attn_bwd(q[r], k[r], v[r], do[r], lse, delta, dq, dk, dv, bd.local.items, bd.local.n,
                         bd.local.segs, softmax_scale=scale)
        grads.append((dq, dk, dv))
        deltas.append(delta)
    for ri, rs in enumerate(sched.rings()):
        members = rs.ring.members
        g = len(members)
        idx = {m: next(j for j, x in enumerate(progs[m].rings) if x.ring_index == ri) for m in members}
        held, gk, gv = {}, {}, {}
        for m in members:
            rp = progs[m].rings[idx[m]]
            pack = devs[m].rings[idx[m]][0]
            rows = max(rp.held_rows)
            buf = torch.zeros(rows, 2, hkv, d, dtype=torch.bfloat16, device=dev)
            n = rp.pack_ranges.shape[0]
            mx = int(rp.pack_ranges[:, 2].max()) if n else 0
            ops.copy_rows(buf[:, 0], k[m], pack, n, mx)
            ops.copy_rows(buf[:, 1], v[m], pack, n, mx)
            held[m] = buf
            gk[m] = torch.zeros(rows, hkv, d, dtype=torch.float32, device=dev)
            gv[m] = torch.zeros(rows, hkv, d, dtype=torch.float32, device=dev)
        for rnd in range(g):
            for m in members:
                rp = progs[m].rings[idx[m]]
                work = bdevs[m].rings[idx[m]][0][rnd]
                n_kv = rp.rounds[rnd].kv_rows
                if work.n:
                    ops.attn_bwd(q[m], held[m][:n_kv, 0], held[m][:n_kv, 1], do[m], outs[m][1], deltas[m],
                                 grads[m][0], gk[m][:n_kv], gv[m][:n_kv], work.items, work.n, work.segs,
                                 softmax_scale=scale)
            nh, nk, nv = {}, {}, {}
            for m in members:
                rp = progs[m].rings[idx[m]]
                n = rp.send_rows(rnd)
                nh[rp.next_rank] = held[m][:n].clone()
                nk[rp.next_rank] = gk[m][:n].clone()
                nv[rp.next_rank] = gv[m][:n].clone()
            held, gk, gv = nh, nk, nv
        for m in members:
            rp = progs[m].rings[idx[m]]
            up = bdevs[m].rings[idx[m]][1]
            n = up.numel() // 3
            mx = int(rp.pack_ranges[:, 2].max()) if n else 0
            if n:
                ops.copy_rows(grads[m][1], gk[m], up, n, mx)
                ops.copy_rows(grads[m][2], gv[m], up, n, mx)
    torch.cuda.synchronize()
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
