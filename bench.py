#!/usr/bin/env python
"""Benchmark of the Zeppelin per-layer hot path on B200s (BASELINE.json metric).

A step = one pass of the hot path over one synthetic batch: host planner
(build_plan + build_schedule + solve_remap + per-rank work lists) -> attention
engine (local varlen kernel + ring rounds over NVLink) -> remap to the linear
layout -> inverse remap.  Prints ONE JSON line on rank 0.

  N = 1: config 2 — Llama-3-8B attention layer (32 Q / 8 KV heads, d128, bf16)
         on a 64K-token github-mixture batch (seed 0), all sequences local.
  N > 1: config 3 — weak scaling, 64K tokens per GPU, one 128K sequence plus a
         github<=128K sample (seed 1), split across GPUs by the planner; ring
         KV exchange over NVLink + remap all-to-allv.

  --impl reference: the layer's CPU path on the host cores: the reference
  package's own planner (baseline/_ref) + torch fp32 SDPA attention of every
  sequence + the remap row moves, whole steps, no extrapolation.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attn+remap layer tokens/s at 1/2/4/8 B200; % of tensor/NVLink roofline"
UNIT = "tokens/s"
FLOP_PER_PAIR = 4 * 128 * 32  # QK^T + PV, forward, d=128, Hq=32
HIDDEN_BYTES = 4096 * 2        # remap row: hidden 4096 bf16


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def workload(n_gpus: int):
    from paper_2509_21841_b200 import workloads as W
    if n_gpus == 1:
        batch = W.c2_batch("github", 0)
        name = "C2: Llama-3-8B attention layer, 64K-token github batch (seed 0), all local, 1 B200"
    else:
        batch = W.c3_batch(n_gpus)
        name = (f"C3: Llama-3-8B attention+remap layer, {65536 * n_gpus}-token long-context mixture "
                f"(128K seq + github<=128K, seed 1), {n_gpus} B200 ring/NVLink")
    return name, batch, W.cluster_for(batch, n_gpus)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: make sure it is sampling
            # before the timed region begins, then drop the idle samples
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- GPU arm

def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_21841_b200 import engine, ops
    from paper_2509_21841_b200 import plan as P, remap as M, schedule as S
    from paper_2509_21841_b200.program import build_rank_program

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ctx = engine.RankContext(rank, world, dev)
    name, batch, cluster = workload(world)
    hq, hkv, d = 32, 8, 128

    stager = engine.TableStager(dev)

    def host_plan():
        plan = P.build_plan(batch, cluster)
        sched = S.build_schedule(plan)
        res = M.solve_remap(plan.tokens_per_rank, M.cost_matrix(cluster))
        prog = build_rank_program(plan, sched, rank, hq, res)
        return plan, sched, prog, engine.DeviceProgram(prog, dev, stager)

    plan, sched, prog, devp = host_plan()
    rows = prog.rows
    lay = prog.remap
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q = torch.randn(rows, hq, d, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(rows, hkv, d, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(rows, hkv, d, device=dev, generator=g, dtype=torch.bfloat16)
    # one activation buffer with max(A_r, B_r) rows: the attention layout is
    # its prefix [0, A_r), the linear layout its prefix [0, B_r); kept rows
    # never move, only the remapped tail crosses NVLink.
    lin_rows = max(lay.linear_rows[rank], rows, 1)
    if world > 1:
        # IPC-shared so peers can read their incoming rows straight out of it
        peer = engine.PeerBuffer(ctx, cluster.token_capacity, hq * d)
        act = peer.buf
    else:
        peer = None
        act = torch.empty(lin_rows, hq * d, device=dev, dtype=torch.bfloat16)
    o = act[:rows].view(rows, hq, d)
    lse = torch.empty(hq, max(rows, 1), device=dev)

    attn_events: list[tuple] = []

    def step(record=False):
        plan_, sched_, prog_, devp_ = host_plan()
        if record:
            ops.set_launch_hook(lambda name, a, b: attn_events.append((name, a, b)))
        engine.attention_forward(plan_, sched_, q, k, v, ctx, prog_, devp_, out=(o, lse))
        ops.set_launch_hook(None)
        if peer is not None:
            # fused remap kernel: peer loads over NVLink, in place
            engine.remap_pull(prog_.remap, peer, act, ctx)
            engine.remap_pull(prog_.remap, peer, act, ctx, inverse=True)
        else:
            yy = engine.remap_forward(prog_.remap, act[:rows], ctx, out=act[:prog_.remap.linear_rows[rank]])
            engine.remap_inverse(prog_.remap, yy, ctx, out=act[:rows])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ops.reset_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record()
        for _ in range(args.steps):
            step(record=True)
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = ops.launch_count()
    ms_local = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total_tokens = batch.total_tokens
    value = total_tokens / (ms / 1e3)

    # dominant kernel: attention launches on this rank inside the timed region
    attn_ms = sum(a.elapsed_time(b) for _, a, b in attn_events) / args.steps
    rank_pairs = prog.pairs_per_head()
    rank_flop = rank_pairs * FLOP_PER_PAIR
    peak, peak_sus, hbm, peak_kind = _peaks()
    achieved = rank_flop / (attn_ms / 1e3) / 1e12 if attn_ms > 0 else 0.0
    stats = torch.tensor([achieved, attn_ms, float(rank_pairs), float(len(attn_events) / args.steps)],
                         device=dev, dtype=torch.float64)
    if world > 1:
        gathered = [torch.zeros_like(stats) for _ in range(world)]
        dist.all_gather(gathered, stats)
    else:
        gathered = [stats]
    per_rank = [x.tolist() for x in gathered]
    busiest = max(range(world), key=lambda i: per_rank[i][2])
    moved = lay.moved_rows()

    remap_stress = None
    if world > 1 and not args.no_remap_stress:
        remap_stress = run_remap_stress(ctx, dev, world, rank, args)

    # end to end through the public API with host buffers (pinned), rank-local
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, dev, rows, hq, hkv, d, host_plan, world, rank)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    # DRAM bytes of this workload's attention launches (busiest rank, one step),
    # measured by ncu for exactly this config (tools/traffic_capture.py)
    traffic, traffic_note = None, "no ncu capture for this N in profiles/r02_attn_traffic.json"
    prof_path = os.path.join(ROOT, "profiles", "r02_attn_traffic.json")
    if os.path.exists(prof_path):
        try:
            cap = json.load(open(prof_path)).get(f"n{world}")
            if cap:
                traffic = cap["dram_bytes_per_step"]
                traffic_note = (f"ncu dram__bytes_read+write of the {cap['launches']} attention launch(es) of one step "
                                f"({cap['workload']}; algorithmic {cap['algorithmic_bytes_per_step']:.3e} B); "
                                "cold-cache serialised capture")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded batch from the reference's length mixtures; N(0,1) q/k/v)",
        "config": {
            "workload": name,
            "total_tokens": total_tokens,
            "sequences": len(batch),
            "heads": [hq, hkv, d],
            "rings": len(plan.ring_groups),
            "remap_rows_moved": moved,
            "l2": "inputs larger than L2 (q/k/v %.0f MB per GPU > 126 MB)" % (rows * (hq + 2 * hkv) * d * 2 / 1e6),
            "parallelism": f"zeppelin plan over {world} GPU(s), one process per GPU",
            "attention_pairs_per_gpu": sum(r[2] for r in per_rank) / world,
            "scaling_note": ("BASELINE config 2 at N=1 (all-local 64K batch); config 3 at N>1 puts a 128K "
                             "sequence in the batch, ~3x the attention pairs per GPU of config 2, so compare "
                             "roofline.aggregate_tflops across N rather than tokens/s"),
        },
        "roofline": {
            "bound": "tensor",
            "achieved": achieved if world == 1 else per_rank[busiest][0],
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": (achieved if world == 1 else per_rank[busiest][0]) / peak,
            "frac_of_sustained": ((achieved if world == 1 else per_rank[busiest][0]) / peak_sus) if peak_sus else None,
            "peak_kind": f"{peak_kind} burst bf16 (MEASURED_PEAKS.json)",
            "traffic": traffic,
            "traffic_note": traffic_note,
            "kernel": "zp_attn_fwd (attn_fwd_kernel)",
            "flop_per_pair": FLOP_PER_PAIR,
            "rank": busiest,
            "rank_pairs": int(per_rank[busiest][2]),
            "attn_ms_per_step": per_rank[busiest][1],
            "aggregate_tflops": sum(r[2] for r in per_rank) * FLOP_PER_PAIR / (ms / 1e3) / 1e12,
            # the step against the slowest rank's attention (ring waits, remap,
            # planner-table uploads are what separate them)
            "attn_ms_max_over_ranks": max(r[1] for r in per_rank),
            "step_over_slowest_attention": ms / max(max(r[1] for r in per_rank), 1e-9),
        },
        "remap_stress": remap_stress,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(batch, cluster, world)
    emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, ctx, dev, rows, hq, hkv, d, host_plan, world, rank):
    """Same metric through the public API (ZeppelinLayer.step_host) with pinned
    HOST q/k/v: every step plans the batch, copies its inputs H2D and reads
    the attention output (after the remap round trip) back D2H; copies of
    neighbouring steps overlap compute on separate streams."""
    import torch
    import torch.distributed as dist

    from paper_2509_21841_b200 import engine

    _, batch, cluster = workload(world)
    layer = engine.ZeppelinLayer(cluster, ctx)
    hq_ = torch.randn(rows, hq, d, dtype=torch.bfloat16).pin_memory()
    hk_ = torch.randn(rows, hkv, d, dtype=torch.bfloat16).pin_memory()
    hv_ = torch.randn(rows, hkv, d, dtype=torch.bfloat16).pin_memory()
    ho_ = [torch.empty(rows, hq, d, dtype=torch.bfloat16).pin_memory() for _ in range(2)]

    def one(i):
        layer.prepare(batch)
        layer.step_host(hq_, hk_, hv_, ho_[i % 2])

    for i in range(max(1, args.warmup)):
        one(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        one(i)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": batch.total_tokens / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": int((hq_.numel() + hk_.numel() + hv_.numel()) * 2),
            "d2h_bytes_per_step": int(ho_[0].numel() * 2),
            "timing": "wall clock over the steps incl. final sync, max over ranks",
            "api": "paper_2509_21841_b200.ZeppelinLayer.prepare + step_host (pipelined H2D / D2H streams)"}


def run_remap_stress(ctx, dev, world, rank, args, total=262144, iters=10):
    """Config 4 (remap alone, hidden 4096 bf16, 256K tokens) on the two
    declared stress layouts of SURVEY 8(d): S1 fan-out (rank 0 holds every
    token) and S2 alternating (even ranks hold 2T/G, odd ranks none).  Both
    the NCCL all-to-allv path and the fused peer-store kernel are timed
    (forward remap, CUDA events, max over ranks); bandwidth is the busiest
    sender's bytes / time against 900 GB/s nominal and 770 GB/s measured
    per-direction NVLink."""
    import torch
    import torch.distributed as dist

    from paper_2509_21841_b200 import engine
    from paper_2509_21841_b200.remap import remap_layout

    hidden = 4096
    out = {}
    layouts = {
        "S1_fan_out": [total] + [0] * (world - 1),
        "S2_alternating": [2 * total // world if i % 2 == 0 else 0 for i in range(world)],
    }
    for name, counts in layouts.items():
        lay = remap_layout(counts)
        a, b = lay.attn_rows[rank], lay.linear_rows[rank]
        sent = [int(lay.matrix[i].sum()) * hidden * 2 for i in range(world)]
        busiest = max(sent)
        res = {"counts": counts, "rows_moved": lay.moved_rows(), "busiest_sender_bytes": busiest}
        # one IPC-shared activation buffer per rank with max(A_i, B_i) rows:
        # the attention layout is its prefix [0, A_i), the linear layout its
        # prefix [0, B_i); kept rows never move, only remapped rows cross NVLink
        act = engine.PeerBuffer(ctx, max(max(lay.attn_rows), max(lay.linear_rows)), hidden)
        act.buf.normal_()
        x, yv = act.buf[:a], act.buf[:b]
        tabs = engine.push_tables(lay, rank, False, dev)
        ptabs = engine.pull_tables(lay, rank, False, dev)
        lay0 = remap_layout([1] * world)  # nothing moves: ready + done kernels only
        tabs0 = engine.push_tables(lay0, rank, False, dev)
        paths = {
            "nccl_all_to_allv": lambda: engine.remap_forward(lay, x, ctx, out=yv),
            "fused_peer_store": lambda: engine.remap_push(lay, x, act, ctx, tables=tabs),
            "fused_peer_load": lambda: engine.remap_pull(lay, act, act.buf, ctx, tables=ptabs),
            "copy_engine_push": lambda: engine.remap_push(lay, x, act, ctx, tables=tabs, copy_engine=True),
            "copy_engine_pull": lambda: engine.remap_pull(lay, act, act.buf, ctx, tables=ptabs, copy_engine=True),
            "handshake_only": lambda: engine.remap_push(lay0, act.buf[:1], act, ctx, tables=tabs0),
        }
        for pname, fn in paths.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            gbs = busiest / (ms / 1e3) / 1e9
            res[pname] = {"ms": ms, "GB_per_s_busiest_sender": gbs, "frac_nvlink_900": gbs / 900.0,
                          "frac_nvlink_770_measured": gbs / 770.0}
        # exactness: every path lands the same rows (rows are overwritten with
        # the same payload each time, the sources never change)
        ref = torch.empty_like(act.buf)
        ref[:b] = engine.remap_forward(lay, x.clone(), ctx)
        same = True
        for pname, fn in paths.items():
            if pname == "handshake_only":
                continue
            act.buf[a:].zero_() if b > a else None
            fn()
            torch.cuda.synchronize()
            same &= bool(torch.equal(act.buf[:b], ref[:b]))
        ok = torch.tensor([int(same)], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        res["all_paths_equal"] = bool(ok.item())
        del act, ref
        torch.cuda.empty_cache()
        out[name] = res
    return out


# ---------------------------------------------------------------------------- CPU arm

def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _reference_package():
    """The UNMODIFIED reference (varlenplan) installed into baseline/_ref
    (pip install --target baseline/_ref /root/reference; travels to the GPU
    box with the snapshot).  None when it is not installed: the bit-exact
    restatement of its planner (paper_2509_21841_b200) is timed instead."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "varlenplan")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import varlenplan
    return varlenplan


class CpuLayer:
    """The layer's CPU path, every rank's work in one process (BASELINE.md
    section 2): the reference's own planner (build_plan + build_schedule +
    solve_remap on the step's batch) and the CPU fp32 torch restatement of
    the work it only counts — causal GQA attention of every sequence
    (scaled_dot_product_attention, enable_gqa; whole sequences: the ring
    rounds compose to exactly this) and the remap row moves (index_select
    along the R3 permutation).  All host threads."""

    def __init__(self, batch, cluster, world: int):
        import numpy as np
        import torch

        from paper_2509_21841_b200 import plan as P, remap as M

        torch.set_num_threads(os.cpu_count() or 1)
        self.batch, self.cluster, self.world = batch, cluster, world
        self.vp = _reference_package()
        if self.vp is not None:
            self.ref_batch = self.vp.SequenceBatch(tuple(batch.sequences))
            c = cluster
            self.ref_cluster = self.vp.ClusterSpec(c.num_nodes, c.gpus_per_node, c.token_capacity,
                                                   c.inv_bw_intra, c.inv_bw_inter)
        g = torch.Generator().manual_seed(0)
        self.seqs = [(sid, n) for sid, n in sorted(batch.sequences, key=lambda x: -x[1])]
        self.qkv = {sid: (torch.randn(1, 32, n, 128, generator=g), torch.randn(1, 8, n, 128, generator=g),
                          torch.randn(1, 8, n, 128, generator=g)) for sid, n in self.seqs}
        plan = P.build_plan(batch, cluster)
        self.lay = M.remap_layout(plan.tokens_per_rank, M.solve_remap(plan.tokens_per_rank, M.cost_matrix(cluster)))
        # remap payload: hidden 4096 fp32 rows per rank (attention layout), and
        # the gather index of every linear-layout row (oracle rule R3)
        from oracle import remap as OR
        src = OR.source_map(list(self.lay.attn_rows), self.lay.matrix)
        self.x = ([torch.randn(n, 4096, generator=g).to(torch.bfloat16) for n in self.lay.attn_rows]
                  if world > 1 else [])  # remap payload: hidden 4096 bf16 rows, as on the GPU
        self.gather = [(torch.from_numpy(np.ascontiguousarray(s[:, 0])), torch.from_numpy(np.ascontiguousarray(s[:, 1])))
                       for s in src] if world > 1 else []
        self.pairs = sum(n * (n + 1) // 2 for _, n in self.seqs)

    def planner(self):
        if self.vp is not None:
            plan = self.vp.build_plan(self.ref_batch, self.ref_cluster)
            self.vp.build_schedule(plan)
            self.vp.solve_remap(list(plan.tokens_per_rank), self.vp.cost_matrix(self.ref_cluster))
        else:
            from paper_2509_21841_b200 import plan as P, remap as M, schedule as S
            plan = P.build_plan(self.batch, self.cluster)
            S.build_schedule(plan)
            M.solve_remap(plan.tokens_per_rank, M.cost_matrix(self.cluster))

    def step(self, limit_tokens: int | None = None) -> dict:
        """One full step (or, for warm-up, attention of the first
        ``limit_tokens`` rows of the shortest sequence).  Returns seconds per
        phase."""
        import torch
        import torch.nn.functional as F

        t0 = time.perf_counter()
        self.planner()
        t1 = time.perf_counter()
        with torch.no_grad():
            for sid, n in (self.seqs if limit_tokens is None else self.seqs[-1:]):
                q, k, v = self.qkv[sid]
                if limit_tokens is not None:
                    m = min(n, limit_tokens)
                    q, k, v = q[:, :, :m], k[:, :, :m], v[:, :, :m]
                F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        t2 = time.perf_counter()
        if limit_tokens is None:
            for j in range(self.world if self.x else 0):
                ranks, rows = self.gather[j]
                out = torch.empty(len(rows), 4096, dtype=torch.bfloat16)
                for r in range(self.world):
                    sel = (ranks == r).nonzero().squeeze(1)
                    if sel.numel():
                        out.index_copy_(0, sel, self.x[r].index_select(0, rows[sel].long()))
        t3 = time.perf_counter()
        return {"planner_s": t1 - t0, "attention_s": t2 - t1, "remap_s": t3 - t2, "total_s": t3 - t0}

    def describe(self, kind: str) -> str:
        planner = ("the reference package itself (varlenplan from baseline/_ref): build_plan + build_schedule + "
                   "solve_remap" if self.vp is not None else
                   "the bit-exact planner restatement (reference not installed): build_plan + build_schedule + "
                   "solve_remap")
        return (f"whole {self.batch.total_tokens}-token batch every step, no extrapolation: {planner}; "
                f"torch fp32 scaled_dot_product_attention(is_causal, enable_gqa) over all {len(self.seqs)} "
                f"sequences ({self.pairs} causal pairs x 32 heads)"
                + ("; remap index_select fwd over all ranks" if self.x else "; remap is a no-op at N=1")
                + f"; {os.cpu_count()} threads on {_cpu_model()}")


def cpu_baseline(batch, cluster, world: int):
    """cpu_baseline field of the GPU arm's line (rank 0, N=1): one full step
    of the CPU path after a short warm-up."""
    cl = CpuLayer(batch, cluster, world)
    cl.step(limit_tokens=512)
    st = cl.step()
    return {"value": batch.total_tokens / st["total_s"], "unit": UNIT, "cores": os.cpu_count() or 1,
            "kind": "port", "sample": cl.describe("baseline"),
            "phases_s": st, "cpu_model": _cpu_model(),
            "attention_tflops": cl.pairs * FLOP_PER_PAIR / st["attention_s"] / 1e12}


def run_reference(args):
    """--impl reference: the CPU path of the same metric and config on the
    host cores (rank 0 only).  Warm-up steps run the planner plus a short
    attention slice; timed steps are whole steps (no extrapolation), at
    least 3 (1 when one step takes over a minute) and then as many of the K
    requested as fit in --ref-budget seconds; the value is the median."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name, batch, cluster = workload(args.gpus)
    cl = CpuLayer(batch, cluster, args.gpus)
    for _ in range(args.warmup):
        cl.step(limit_tokens=512)
    steps = []
    t_start = time.perf_counter()
    for i in range(args.steps):
        steps.append(cl.step())
        # at least 3 whole steps, or 1 when a single step already takes a
        # minute (config 3 at N=8 is ~2.5 min of CPU attention per step)
        need = 3 if steps[0]["total_s"] < 60.0 else 1
        if len(steps) >= need and time.perf_counter() - t_start > args.ref_budget:
            break
    med = statistics.median(s["total_s"] for s in steps)
    value = batch.total_tokens / med
    phases = {k: statistics.median(s[k] for s in steps) for k in steps[0]}
    emit({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (same batch as the GPU arm; N(0,1) fp32 q/k/v)",
        "impl": "reference",
        "config": {"workload": name, "total_tokens": batch.total_tokens, "sequences": len(batch)},
        "steps_timed": len(steps), "phases_s_median": phases,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count() or 1,
                         "kind": "port", "sample": cl.describe("reference"),
                         "cpu_model": _cpu_model(),
                         "attention_tflops": cl.pairs * FLOP_PER_PAIR / phases["attention_s"] / 1e12},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


_JSON_OUT = None


def emit(line: dict) -> None:
    """Print the single JSON result line on the ORIGINAL stdout (library
    banners, e.g. NCCL's version line, are routed to stderr)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def run_block(args):
    """Config 5: full Llama-3-8B block (norm, QKV, remap, RoPE, attention,
    remap, O, norm, SwiGLU MLP) on the 256K-token github<=128K batch (seed 1)
    over N GPUs; tokens/s of the whole block, same JSON contract."""
    import torch
    import torch.distributed as dist

    from paper_2509_21841_b200 import block as B, engine, ops
    from paper_2509_21841_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ctx = engine.RankContext(rank, world, dev)
    batch = W.c4_batch()
    cluster = W.cluster_for(batch, world)
    w = B.BlockWeights.random(dev, seed=0)
    blk = B.ZeppelinBlock(cluster, w, ctx, max_pos=262144)
    blk.prepare(batch)
    a, b = blk.rows
    x = torch.randn(b, B.HIDDEN, device=dev, dtype=torch.bfloat16)

    def step():
        blk.prepare(batch)
        return blk.forward(x)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ops.reset_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    gemm, attn = blk.flops_per_step()
    fl = torch.tensor([float(gemm), float(attn)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(fl)
    peak, peak_sus, _, kind = _peaks()
    total_tf = float(fl.sum()) / (ms / 1e3) / 1e12
    line = {
        "metric": "full transformer block tokens/s (config 5)", "value": batch.total_tokens / (ms / 1e3),
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init Llama-3-8B block weights, N(0,1) hidden states)",
        "config": {"workload": "C5: Llama-3-8B block, 256K-token github<=128K batch (seed 1)",
                   "total_tokens": batch.total_tokens, "rings": len(blk.plan.ring_groups),
                   "remap_rows_moved": int(blk.layout.moved_rows()),
                   "gemms": "cuBLAS bf16 (torch.matmul/addmm)"},
        "tflops_aggregate": total_tf, "tflops_per_gpu": total_tf / world,
        "frac_of_peak_per_gpu": total_tf / world / peak, "gemm_flop": float(fl[0]), "attn_flop": float(fl[1]),
        "gpu_launches": ops.launch_count(), "clocks": clocks.summary(),
    }
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_backward(args):
    """one training step of the attention layer — forward
    (LocalTask + ring rounds) and backward (zp_attn_bwd, ring dK/dV travelling
    with the KV sets) — on the layer workload (C2 at N=1, C3 at N>1)."""
    import torch
    import torch.distributed as dist

    from paper_2509_21841_b200 import engine, ops
    from paper_2509_21841_b200 import plan as P, schedule as S
    from paper_2509_21841_b200.program import build_bwd_program, build_rank_program

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ctx = engine.RankContext(rank, world, dev)
    name, batch, cluster = workload(world)
    hq, hkv, d = 32, 8, 128
    plan = P.build_plan(batch, cluster)
    sched = S.build_schedule(plan)
    prog = build_rank_program(plan, sched, rank, hq)
    devp = engine.DeviceProgram(prog, dev)
    bdev = engine.BwdDeviceProgram(build_bwd_program(prog, hkv), dev)
    rows = prog.rows
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    q, dout = (torch.randn(rows, hq, d, device=dev, generator=g, dtype=torch.bfloat16) for _ in range(2))
    k, v = (torch.randn(rows, hkv, d, device=dev, generator=g, dtype=torch.bfloat16) for _ in range(2))
    events: list[tuple] = []

    def step(record=False):
        if record:
            ops.set_launch_hook(lambda nm, a, b: events.append((nm, a, b)))
        o, lse = engine.attention_forward(plan, sched, q, k, v, ctx, prog, devp)
        engine.attention_backward(plan, sched, q, k, v, o, lse, dout, ctx, prog, bdev)
        ops.set_launch_hook(None)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ops.reset_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(args.steps):
            step(record=True)
        e1.record()
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    fwd_ms = sum(a.elapsed_time(b) for nm, a, b in events if nm == "zp_attn_fwd") / args.steps
    bwd_ms = sum(a.elapsed_time(b) for nm, a, b in events if nm == "zp_attn_bwd") / args.steps
    pairs = prog.pairs_per_head()
    st = torch.tensor([float(pairs), fwd_ms, bwd_ms], device=dev, dtype=torch.float64)
    if world > 1:
        gathered = [torch.zeros_like(st) for _ in range(world)]
        dist.all_gather(gathered, st)
    else:
        gathered = [st]
    per = [x.tolist() for x in gathered]
    busiest = max(range(world), key=lambda i: per[i][0])
    peak, peak_sus, _, kind = _peaks()
    bwd_flop = per[busiest][0] * 10 * 128 * 32
    bwd_tf = bwd_flop / (per[busiest][2] / 1e3) / 1e12 if per[busiest][2] > 0 else 0.0
    fwd_tf = per[busiest][0] * FLOP_PER_PAIR / (per[busiest][1] / 1e3) / 1e12 if per[busiest][1] > 0 else 0.0
    line = {
        "metric": "attention layer training step (fwd+bwd) tokens/s", "value": batch.total_tokens / (ms / 1e3),
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded batch from the reference's length mixtures; N(0,1) q/k/v/dO)",
        "config": {"workload": name, "total_tokens": batch.total_tokens, "rings": len(plan.ring_groups)},
        "roofline": {"bound": "tensor", "kernel": "zp_attn_bwd (attn_bwd_kernel)", "achieved": bwd_tf,
                     "peak": peak, "unit": "TFLOP/s", "frac": bwd_tf / peak,
                     "flop_per_pair": 10 * 128 * 32, "rank": busiest, "bwd_ms_per_step": per[busiest][2],
                     "fwd_ms_per_step": per[busiest][1], "fwd_tflops": fwd_tf,
                     "peak_kind": f"{kind} burst bf16 (MEASURED_PEAKS.json)"},
        "gpu_launches": ops.launch_count(), "clocks": clocks.summary(),
    }
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_compare(args):
    """the paper's comparison executed, not modelled.  The
    same batch runs under zeppelin, te_cp, llama_cp and hybrid_dp plans
    (reference baselines.py) on the same GPUs; per strategy the full Llama-3-8B
    block (config 5 code path) and its attention+remap part are timed."""
    import torch
    import torch.distributed as dist

    from paper_2509_21841_b200 import block as B, engine, ops
    from paper_2509_21841_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ctx = engine.RankContext(rank, world, dev)
    batch = W.c4_batch()  # 256K-token long-tailed github<=128K batch (configs 4/5)
    cluster = W.cluster_for(batch, world)
    w = B.BlockWeights.random(dev, seed=0)
    results = {}
    for strategy in ("zeppelin", "te_cp", "llama_cp", "hybrid_dp"):
        try:
            blk = B.ZeppelinBlock(cluster, w, ctx, max_pos=262144, strategy=strategy)
            blk.prepare(batch)
        except Exception as exc:  # e.g. InfeasibleBatch under the even split
            results[strategy] = {"error": f"{type(exc).__name__}: {exc}"}
            continue
        a, b = blk.rows
        x = torch.randn(b, B.HIDDEN, device=dev, dtype=torch.bfloat16)
        q = torch.randn(a, 32, 128, device=dev, dtype=torch.bfloat16)
        k = torch.randn(a, 8, 128, device=dev, dtype=torch.bfloat16)
        v = torch.randn(a, 8, 128, device=dev, dtype=torch.bfloat16)
        o = torch.empty_like(q)
        lse = torch.empty(32, max(a, 1), device=dev)
        kvx = "allgather" if strategy == "llama_cp" else "ring"

        def attn_step():
            engine.attention_forward(blk.plan, blk.schedule, q, k, v, ctx, blk.program, blk.device_program,
                                     out=(o, lse), kv_exchange=kvx)
            if blk.peer_o is not None:
                blk.peer_o.buf[:a].copy_(o.view(a, -1))
                engine.remap_pull(blk.layout, blk.peer_o, blk.peer_o.buf, ctx)
                engine.remap_pull(blk.layout, blk.peer_o, blk.peer_o.buf, ctx, inverse=True)

        res = {"rows_per_rank_max": max(blk.plan.tokens_per_rank), "rings": len(blk.plan.ring_groups)}
        for name, fn in (("attention_layer", attn_step), ("block", lambda: blk.forward(x))):
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            res[name] = {"ms": ms, "tokens_per_s": batch.total_tokens / (ms / 1e3)}
        results[strategy] = res
        del blk, q, k, v, o, x
        torch.cuda.empty_cache()
    z = results.get("zeppelin", {})
    for sname, r in results.items():
        if "error" not in r and "error" not in z:
            r["zeppelin_speedup_block"] = r["block"]["ms"] / z["block"]["ms"]
            r["zeppelin_speedup_attention_layer"] = r["attention_layer"]["ms"] / z["attention_layer"]["ms"]
    if rank == 0:
        emit({"metric": "strategy comparison (block and attention+remap ms, max over ranks)",
              "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
              "config": {"workload": "C4/C5 batch: 256K-token github<=128K (seed 1)", "total_tokens": batch.total_tokens,
                         "sequences": len(batch)}, "results": results})
    if world > 1:
        dist.destroy_process_group()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)  # everything else written to fd 1 (C libraries included) goes to stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["zeppelin", "reference"], default="zeppelin")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="--impl reference: stop timing whole steps after this many seconds (>= 3 steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-remap-stress", action="store_true")
    ap.add_argument("--workload", choices=["layer", "c5", "compare", "train"], default="layer",
                    help="layer: attn+remap (BASELINE metric); c5: full transformer block; "
                         "train: attention fwd+bwd step")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "zeppelin":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5":
        run_block(args)
    elif args.workload == "compare":
        run_compare(args)
    elif args.workload == "train":
        run_backward(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
