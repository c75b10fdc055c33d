"""Run every rank of a plan in ONE process on ONE GPU (sequentially).

Used to validate the ring programs with the real sm_100a kernels when only
one B200 is available: each emulated rank packs its KV set, runs its rounds
with ``zp_attn_fwd`` and hands its buffer to the next ring position with a
device copy instead of NCCL.  No kernel ever waits on another (launches are
serialised on one stream).
"""

from __future__ import annotations

import math

import torch

from . import ops
from .engine import DeviceProgram
from .program import build_rank_program


def gather_rank(seq_tensors: dict, plan, rank: int, device) -> torch.Tensor:
    parts = [seq_tensors[f.sequence_id][f.start:f.end] for f in plan.fragments[rank]]
    return torch.cat(parts, 0).to(device).contiguous()


def emulate_ranks_on_one_gpu(plan, sched, sq: dict, sk: dict, sv: dict, device="cuda"):
    hq = next(iter(sq.values())).shape[1]
    hkv, d = next(iter(sk.values())).shape[1:]
    scale = 1.0 / math.sqrt(d)
    progs = [build_rank_program(plan, sched, r, hq) for r in range(plan.num_ranks)]
    devs = [DeviceProgram(p, torch.device(device)) for p in progs]
    q = [gather_rank(sq, plan, r, device) for r in range(plan.num_ranks)]
    k = [gather_rank(sk, plan, r, device) for r in range(plan.num_ranks)]
    v = [gather_rank(sv, plan, r, device) for r in range(plan.num_ranks)]
    outs = []
    for r, (p, dp) in enumerate(zip(progs, devs)):
        o = torch.zeros_like(q[r])
        lse = torch.full((hq, max(p.rows, 1)), float("-inf"), device=device)
        if dp.local.n:
            ops.attn_fwd(q[r], k[r], v[r], dp.local.items, dp.local.n, dp.local.segs, o, lse, softmax_scale=scale)
        outs.append((o, lse))
    for ri, rs in enumerate(sched.rings()):
        members = rs.ring.members
        g = len(members)
        idx = {m: next(j for j, x in enumerate(progs[m].rings) if x.ring_index == ri) for m in members}
        held, state = {}, {}
        for m in members:
            rp = progs[m].rings[idx[m]]
            pack = devs[m].rings[idx[m]][0]
            buf = torch.zeros(max(rp.held_rows), 2, hkv, d, dtype=torch.bfloat16, device=device)
            n = rp.pack_ranges.shape[0]
            mx = int(rp.pack_ranges[:, 2].max()) if n else 0
            ops.copy_rows(buf[:, 0], k[m], pack, n, mx)
            ops.copy_rows(buf[:, 1], v[m], pack, n, mx)
            held[m] = buf
            rows = max(rp.state_rows, 1)
            state[m] = (torch.zeros(rows, hq, d, device=device), torch.zeros(2, hq, rows, device=device))
        for rnd in range(g):
            for m in members:
                rp = progs[m].rings[idx[m]]
                work = devs[m].rings[idx[m]][1][rnd]
                n_kv = rp.rounds[rnd].kv_rows
                if work.n:
                    ops.attn_fwd(q[m], held[m][:n_kv, 0], held[m][:n_kv, 1], work.items, work.n, work.segs,
                                 outs[m][0], outs[m][1], state[m][0], state[m][1], softmax_scale=scale)
            if rnd < g - 1:
                nxt = {}
                for m in members:
                    rp = progs[m].rings[idx[m]]
                    nxt[rp.next_rank] = held[m][:rp.send_rows(rnd)].clone()
                held = nxt
    torch.cuda.synchronize()
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
