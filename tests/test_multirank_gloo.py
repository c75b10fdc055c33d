"""World-size-2 host path over gloo on CPU: ring KV exchange bookkeeping and
the remap all-to-allv slices, with the kernel replaced by the oracle's
work-item interpreter (test-only).  The ring hops follow the executor's pull
plan (RingProgram.hops: buffer indices and row counts), with each pull of
hop r carried by a gloo send/recv pair instead of a copy-engine read."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import attention as OA
from oracle import remap as OR
from oracle import worklist as OW
from paper_2509_21841_b200 import plan as P, schedule as S, workloads as W
from paper_2509_21841_b200.batch import SequenceBatch
from paper_2509_21841_b200.cluster import ClusterSpec
from paper_2509_21841_b200.program import build_rank_program


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, lengths, cap, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hq, hkv, d = 4, 2, 16
        plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), ClusterSpec(1, world, cap, 1.0, 1.0))
        sched = S.build_schedule(plan)
        rng = np.random.default_rng(0)  # same draws on every rank
        seqs = sorted(plan.sequence_lengths.items())
        sq = {s: rng.standard_normal((n, hq, d)) for s, n in seqs}
        sk = {s: rng.standard_normal((n, hkv, d)) for s, n in seqs}
        sv = {s: rng.standard_normal((n, hkv, d)) for s, n in seqs}
        pr = build_rank_program(plan, sched, rank, hq)
        q, k, v = (OA.gather_rank(x, plan, rank) for x in (sq, sk, sv))
        o = np.zeros((pr.rows, hq, d))
        lse = np.full((hq, pr.rows), -np.inf)
        OW.run_items(pr.local.items, pr.local.segs, q, k, v, o, lse, None, d ** -0.5)
        for rp in pr.rings:
            rows = max(rp.held_rows)
            nb = rp.n_buffers
            hops = rp.hops()
            bufs = [torch.zeros(rows, 2, hkv, d, dtype=torch.float64) for _ in range(nb)]
            for dst, src, cnt in rp.pack_ranges:
                bufs[0][dst:dst + cnt, 0] = torch.from_numpy(k[src:src + cnt])
                bufs[0][dst:dst + cnt, 1] = torch.from_numpy(v[src:src + cnt])
            st = OW.State(max(rp.state_rows, 1), hq, d)
            for r in range(rp.group_size):
                rr = rp.rounds[r]
                kv = bufs[r % nb][:rr.kv_rows].numpy()
                OW.run_items(rr.work.items, rr.work.segs, q, kv[:, 0], kv[:, 1], o, lse, st, d ** -0.5)
                if r < rp.group_size - 1:
                    h = hops[r]
                    # successor pulls my src_buf (same index on every position); I pull the predecessor's
                    ops = []
                    if rp.send_rows(r):
                        ops.append(dist.P2POp(dist.isend, bufs[h.src_buf][:rp.send_rows(r)].contiguous(),
                                              rp.next_rank))
                    if h.rows:
                        ops.append(dist.P2POp(dist.irecv, bufs[h.dst_buf][:h.rows], rp.prev_rank))
                    if ops:
                        for req in dist.batch_isend_irecv(ops):
                            req.wait()
        ref, _ = OA.run_plan(plan, sched, sq, sk, sv, d ** -0.5)
        err_attn = float(np.abs(o - ref[rank][0]).max())
        # remap forward / inverse over gloo with the executor's slices
        lay = pr.remap
        # payload = (rank, row) ids: the row permutation must be exact
        x = torch.stack([torch.full((pr.rows,), float(rank), dtype=torch.float64),
                         torch.arange(pr.rows, dtype=torch.float64)], dim=1)
        kept, (s0, s1), (r0, r1), send, recv = lay.forward_slices(rank)
        y = torch.zeros(lay.linear_rows[rank], x.shape[1], dtype=x.dtype)
        y[:kept] = x[:kept]
        dist.all_to_all_single(y[r0:r1], x[s0:s1].contiguous(), output_split_sizes=recv, input_split_sizes=send)
        want = OR.source_map(list(lay.attn_rows), lay.matrix)[rank]
        err_fwd = float(np.abs(y.numpy() - want).max())
        kept, (s0, s1), (r0, r1), send, recv = lay.inverse_slices(rank)
        back = torch.zeros_like(x)
        back[:kept] = y[:kept]
        dist.all_to_all_single(back[r0:r1], y[s0:s1].contiguous(), output_split_sizes=recv, input_split_sizes=send)
        results[rank] = (err_attn, err_fwd, float((back - x).abs().max()), len(pr.rings))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("lengths,cap", [([66, 73, 306, 41, 169, 241, 53, 37], 497),
                                         ([700, 30, 200, 90], 540)])
def test_two_rank_ring_and_remap_over_gloo(lengths, cap):
    world = 2
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), lengths, cap, results), nprocs=world, join=True)
        res = dict(results)
    assert sorted(res) == [0, 1]
    for rank, (ea, ef, eb, nrings) in res.items():
        assert nrings >= 1
        assert ea < 1e-10 and ef == 0.0 and eb == 0.0, res
