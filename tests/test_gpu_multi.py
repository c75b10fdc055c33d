"""Multi-GPU executor (NCCL ring exchange + all-to-allv remap), one process per
GPU, against the fp64 oracle.  Needs >= 2 B200s; skipped otherwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, lengths, results):
    import torch.distributed as dist
    from oracle import attention as OA
    from oracle import remap as OR
    from paper_2509_21841_b200 import engine, plan as P, schedule as S, remap as M
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import single_box
    from paper_2509_21841_b200.emulate import gather_rank

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        batch = SequenceBatch(tuple(enumerate(lengths)))
        cluster = single_box(world, batch.total_tokens)
        plan = P.build_plan(batch, cluster)
        sched = S.build_schedule(plan)
        g = torch.Generator().manual_seed(1)
        seqs = sorted(plan.sequence_lengths.items())
        sq = {s: torch.randn(n, 32, 128, generator=g).to(torch.bfloat16) for s, n in seqs}
        sk = {s: torch.randn(n, 8, 128, generator=g).to(torch.bfloat16) for s, n in seqs}
        sv = {s: torch.randn(n, 8, 128, generator=g).to(torch.bfloat16) for s, n in seqs}
        ctx = engine.RankContext(rank, world)
        q, k, v = (gather_rank(x, plan, rank, "cuda") for x in (sq, sk, sv))
        o, lse = engine.attention_forward(plan, sched, q, k, v, ctx)
        lay = M.remap_layout(plan.tokens_per_rank, M.solve_remap(plan.tokens_per_rank, M.cost_matrix(cluster)))
        ids = torch.stack([torch.full((q.shape[0],), rank, dtype=torch.int32),
                           torch.arange(q.shape[0], dtype=torch.int32)], 1)
        ids = torch.cat([ids, torch.zeros(q.shape[0], 2, dtype=torch.int32)], 1).cuda()  # 16-byte rows
        y = engine.remap_forward(lay, ids, ctx)
        back = engine.remap_inverse(lay, y, ctx)
        # fused peer-store path (CUDA IPC landing buffers), twice to exercise epochs
        lin = engine.PeerBuffer(ctx, max(lay.linear_rows), 4, torch.int32)
        att = engine.PeerBuffer(ctx, max(lay.attn_rows), 4, torch.int32)
        push_ok = True
        for it in range(2):
            att.buf[:q.shape[0]].copy_(ids)
            yp = engine.remap_push(lay, att.buf[:q.shape[0]], lin, ctx)
            torch.cuda.synchronize()
            push_ok &= bool(torch.equal(yp, y))
            yp[:, 2] = it + 7  # scribble, then bring the rows home
            bp = engine.remap_push(lay, yp, att, ctx, inverse=True)
            torch.cuda.synchronize()
            push_ok &= bool(torch.equal(bp[:, :2], ids[:, :2])) and bool((bp[:, 2] == it + 7).all())
        # the layer API: attention into the IPC activation buffer + fused pull remap
        layer = engine.ZeppelinLayer(cluster, ctx)
        layer.prepare(batch)
        lo, llse, ly = layer.forward(q, k, v)
        o_copy = lo.clone()
        lx = layer.backward_layout(ly)
        torch.cuda.synchronize()
        layer_ok = bool(torch.equal(lx.view_as(o_copy), o_copy)) and bool(torch.equal(o_copy, o))
        f64 = lambda m: {s: t.double().numpy() for s, t in m.items()}  # noqa: E731
        ref, _ = OA.run_plan(plan, sched, f64(sq), f64(sk), f64(sv), 128 ** -0.5)
        err = float(np.abs(o.float().cpu().numpy() - ref[rank][0]).max()) if q.shape[0] else 0.0
        want = OR.source_map(list(lay.attn_rows), lay.matrix)[rank]
        perm_ok = bool(np.array_equal(y[:, :2].cpu().numpy(), want))
        back_ok = bool(torch.equal(back, ids))
        results[rank] = (err, perm_ok, back_ok and push_ok and layer_ok, len(plan.ring_groups))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("lengths", [[3000, 300, 1200, 40, 700], [4000, 1000, 900, 64]])
def test_multi_gpu_attention_and_remap(lengths):
    world = min(torch.cuda.device_count(), 4)
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_worker, args=(world, _port(), lengths, res), nprocs=world, join=True)
        res = dict(res)
    assert sorted(res) == list(range(world))
    for rank, (err, perm_ok, back_ok, nrings) in res.items():
        assert err <= 2e-2 and perm_ok and back_ok, res


def _block_worker(rank, world, port, lengths, results):
    import torch.distributed as dist
    from paper_2509_21841_b200 import block as B, engine
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import single_box

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        batch = SequenceBatch(tuple(enumerate(lengths)))
        cluster = single_box(world, batch.total_tokens)
        w = B.BlockWeights.random("cuda", seed=3)
        blk = B.ZeppelinBlock(cluster, w, engine.RankContext(rank, world), max_pos=8192)
        plan = blk.prepare(batch)
        g = torch.Generator(device="cuda").manual_seed(5)
        x_seq = {s: torch.randn(n, 4096, device="cuda", generator=g).to(torch.bfloat16)
                 for s, n in enumerate(lengths)}
        toks = B.linear_tokens(plan, blk.layout, rank)
        x = torch.stack([x_seq[int(s)][int(p)] for s, p in toks])
        out = blk.forward(x)
        out2 = blk.forward(x)  # second pass exercises the remap epochs
        torch.cuda.synchronize()
        ref = B.reference_block(x_seq, w)
        want = torch.stack([ref[int(s)][int(p)] for s, p in toks])
        err = (out.float() - want).abs()
        scale = want.abs().max().item()
        results[rank] = (err.max().item() / scale, err.mean().item() / scale, bool(torch.equal(out, out2)),
                         len(plan.ring_groups), int(blk.layout.moved_rows()))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_full_block_matches_fp32_reference():
    world = min(torch.cuda.device_count(), 4)
    lengths = [2500, 300, 700, 90, 1000]
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_block_worker, args=(world, _port(), lengths, res), nprocs=world, join=True)
        res = dict(res)
    assert sorted(res) == list(range(world))
    assert any(v[3] > 0 for v in res.values()), "config must exercise rings"
    for rank, (emax, emean, same, nr, moved) in res.items():
        assert emax <= 3e-2 and emean <= 3e-3 and same, res


def _strategy_worker(rank, world, port, lengths, results):
    import torch.distributed as dist
    from oracle import attention as OA
    from paper_2509_21841_b200 import engine, schedule as S
    from paper_2509_21841_b200.baselines import plan_for
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import single_box
    from paper_2509_21841_b200.emulate import gather_rank

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        batch = SequenceBatch(tuple(enumerate(lengths)))
        cluster = single_box(world, batch.total_tokens, slack=1.5)
        g = torch.Generator().manual_seed(2)
        seqs = sorted(batch.lengths.items())
        sq = {s: torch.randn(n, 8, 128, generator=g).to(torch.bfloat16) for s, n in seqs}
        sk = {s: torch.randn(n, 2, 128, generator=g).to(torch.bfloat16) for s, n in seqs}
        sv = {s: torch.randn(n, 2, 128, generator=g).to(torch.bfloat16) for s, n in seqs}
        f64 = lambda m: {s: t.double().numpy() for s, t in m.items()}  # noqa: E731
        out = {}
        for strategy in ("te_cp", "llama_cp", "hybrid_dp"):
            plan = plan_for(strategy, batch, cluster)
            sched = S.build_schedule(plan)
            q, k, v = (gather_rank(x, plan, rank, "cuda") for x in (sq, sk, sv))
            o, lse = engine.attention_forward(plan, sched, q, k, v, engine.RankContext(rank, world),
                                              kv_exchange="allgather" if strategy == "llama_cp" else "ring")
            torch.cuda.synchronize()
            ref, _ = OA.run_plan(plan, sched, f64(sq), f64(sk), f64(sv), 128 ** -0.5)
            out[strategy] = float(np.abs(o.float().cpu().numpy() - ref[rank][0]).max()) if q.shape[0] else 0.0
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_comparison_strategies_execute_exactly():
    world = min(torch.cuda.device_count(), 4)
    lengths = [3000, 40, 700, 1200, 90]
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_strategy_worker, args=(world, _port(), lengths, res), nprocs=world, join=True)
        res = dict(res)
    assert sorted(res) == list(range(world))
    for rank, errs in res.items():
        for strategy, err in errs.items():
            assert err <= 2e-2, (rank, strategy, err)


def _backward_worker(rank, world, port, lengths, results):
    import torch.distributed as dist
    from paper_2509_21841_b200 import engine, plan as P, schedule as S
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import single_box
    from paper_2509_21841_b200.emulate import gather_rank

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        batch = SequenceBatch(tuple(enumerate(lengths)))
        plan = P.build_plan(batch, single_box(world, batch.total_tokens))
        sched = S.build_schedule(plan)
        g = torch.Generator().manual_seed(4)
        seqs = sorted(plan.sequence_lengths.items())
        mk = lambda h: {s: torch.randn(n, h, 128, generator=g).to(torch.bfloat16) for s, n in seqs}  # noqa: E731
        sq, sk, sv, sdo = mk(32), mk(8), mk(8), mk(32)
        ctx = engine.RankContext(rank, world)
        q, k, v, do = (gather_rank(x, plan, rank, "cuda") for x in (sq, sk, sv, sdo))
        o, lse = engine.attention_forward(plan, sched, q, k, v, ctx)
        dq, dk, dv = engine.attention_backward(plan, sched, q, k, v, o, lse, do, ctx)
        torch.cuda.synchronize()
        # fp32 autograd of whole sequences, sliced to this rank's fragments
        ref = {}
        for s, n in seqs:
            qf, kf, vf = (t[s].float().cuda().requires_grad_(True) for t in (sq, sk, sv))
            out = torch.nn.functional.scaled_dot_product_attention(
                qf.transpose(0, 1), kf.repeat_interleave(4, 1).transpose(0, 1),
                vf.repeat_interleave(4, 1).transpose(0, 1), is_causal=True).transpose(0, 1)
            out.backward(sdo[s].float().cuda())
            ref[s] = (qf.grad, kf.grad, vf.grad)
        worst = 0.0
        for j, got in enumerate((dq, dk, dv)):
            want = torch.cat([ref[f.sequence_id][j][f.start:f.end] for f in plan.fragments[rank]])
            err = (got.float() - want).abs().max().item()
            worst = max(worst, err / (want.abs().max().item() + 1e-6))
        results[rank] = (worst, len(plan.ring_groups))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_backward_with_ring_dkv_exchange():
    world = min(torch.cuda.device_count(), 4)
    lengths = [3000, 300, 1200, 40, 700]
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_backward_worker, args=(world, _port(), lengths, res), nprocs=world, join=True)
        res = dict(res)
    assert sorted(res) == list(range(world))
    assert any(v[1] > 0 for v in res.values()), "config must exercise rings"
    for rank, (rel, _) in res.items():
        assert rel <= 2.5e-2, res


def _host_fed_worker(rank, world, port, results):
    """ZeppelinLayer.step_host (pinned host inputs, per-step planning with the
    work lists and both remap tables staged through reused slots, H2D / D2H
    streams) over back-to-back steps with DIFFERENT batches: every step's
    output equals the device path for that batch (no staged table or slot is
    overwritten while a step that reads it is in flight)."""
    import torch.distributed as dist
    from paper_2509_21841_b200 import engine
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import single_box

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        lens = [[3000, 300, 1200, 40, 700], [700, 40, 1200, 300, 3000], [2000, 2000, 1000, 200, 40],
                [5000, 100, 80, 40, 20], [1240, 1000, 1000, 1000, 1000]]
        batches = [SequenceBatch(tuple(enumerate(x))) for x in lens]
        cluster = single_box(world, batches[0].total_tokens)
        ctx = engine.RankContext(rank, world)
        layer = engine.ZeppelinLayer(cluster, ctx)
        g = torch.Generator().manual_seed(rank)
        ins, outs = [], []
        for b in batches:
            layer.prepare(b)
            rows = layer.program.rows
            qkv = tuple(torch.randn(rows, h, 128, generator=g).to(torch.bfloat16).pin_memory() for h in (32, 8, 8))
            ins.append(qkv)
            outs.append(torch.empty(rows, 32, 128, dtype=torch.bfloat16).pin_memory())
        for i, b in enumerate(batches):
            layer.prepare(b)
            layer.step_host(*ins[i], outs[i])
        torch.cuda.synchronize()
        ok = True
        for i, b in enumerate(batches):
            layer.prepare(b)
            o, _ = layer.attention(*(x.cuda() for x in ins[i]))
            torch.cuda.synchronize()
            ok &= bool(torch.equal(outs[i], o.cpu()))
        results[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_host_fed_steps_with_varying_batches():
    world = min(torch.cuda.device_count(), 4)
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_host_fed_worker, args=(world, _port(), res), nprocs=world, join=True)
        res = dict(res)
    assert sorted(res) == list(range(world)) and all(res.values()), res
