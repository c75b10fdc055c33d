"""Per-rank programs (work lists, ring buffers, exchange peers, remap slices)
interpreted on the CPU against the oracle — the host half of the executor."""
import json
import os

import numpy as np
import pytest

from oracle import attention as OA
from oracle import remap as OR
from oracle import worklist as OW
from paper_2509_21841_b200 import plan as P, schedule as S, remap as M, workloads as W
from paper_2509_21841_b200.batch import SequenceBatch
from paper_2509_21841_b200.cluster import ClusterSpec
from paper_2509_21841_b200.program import build_rank_program


def simulate(plan, hq=4, hkv=2, d=16, seed=0):
    """Run every rank's program with an in-process ring exchange."""
    sched = S.build_schedule(plan)
    lengths = sorted(plan.sequence_lengths.items())
    rng = np.random.default_rng(seed)
    sq = {s: rng.standard_normal((n, hq, d)) for s, n in lengths}
    sk = {s: rng.standard_normal((n, hkv, d)) for s, n in lengths}
    sv = {s: rng.standard_normal((n, hkv, d)) for s, n in lengths}
    progs = [build_rank_program(plan, sched, r, hq) for r in range(plan.num_ranks)]
    q = [OA.gather_rank(sq, plan, r) for r in range(plan.num_ranks)]
    k = [OA.gather_rank(sk, plan, r) for r in range(plan.num_ranks)]
    v = [OA.gather_rank(sv, plan, r) for r in range(plan.num_ranks)]
    outs = []
    for r, pr in enumerate(progs):
        n = pr.rows
        o = np.zeros((n, hq, d))
        lse = np.full((hq, n), -np.inf)
        if n:
            OW.run_items(pr.local.items, pr.local.segs, q[r], k[r], v[r], o, lse, None, d ** -0.5)
        outs.append((o, lse))
    # rings in global order; each member packs, then KV rotates i -> i+1
    for ri, rs in enumerate(sched.rings()):
        members = rs.ring.members
        g = len(members)
        rp = {m: next(x for x in progs[m].rings if x.ring_index == ri) for m in members}
        held = {}
        for m in members:
            p = rp[m]
            buf = np.zeros((max(p.held_rows), 2, hkv, d))
            for dst, src, cnt in p.pack_ranges:
                buf[dst:dst + cnt, 0] = k[m][src:src + cnt]
                buf[dst:dst + cnt, 1] = v[m][src:src + cnt]
            held[m] = buf
        states = {m: OW.State(max(rp[m].state_rows, 1), hq, d) for m in members}
        for rnd in range(g):
            for m in members:
                p = rp[m]
                rr = p.rounds[rnd]
                kv = held[m][:rr.kv_rows]
                OW.run_items(rr.work.items, rr.work.segs, q[m], kv[:, 0], kv[:, 1], *outs[m], states[m], d ** -0.5)
            if rnd < g - 1:
                nxt = {}
                for m in members:
                    p = rp[m]
                    assert p.send_rows(rnd) == rp[p.next_rank].recv_rows(rnd)
                    nxt[p.next_rank] = held[m][:p.send_rows(rnd)].copy()
                held = nxt
    return sched, outs, (sq, sk, sv)


def check(plan, **kw):
    sched, outs, (sq, sk, sv) = simulate(plan, **kw)
    d = next(iter(sq.values())).shape[2]
    ref, _ = OA.run_plan(plan, sched, sq, sk, sv, d ** -0.5)
    for (o, l), (ro, rl) in zip(outs, ref):
        assert np.abs(o - ro).max() < 1e-10
        assert np.abs(l - rl).max() < 1e-10


def test_c1_program_matches_oracle():
    check(P.build_plan(W.c1_batch(), W.c1_cluster()))


@pytest.mark.parametrize("seed", range(8))
def test_random_plans_program_matches_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    g = int(rng.choice([2, 3, 4, 5]))
    lengths = [int(x) for x in rng.integers(1, 400, size=int(rng.integers(2, 9)))]
    lengths[int(rng.integers(len(lengths)))] = int(rng.integers(300, 900))
    total = sum(lengths)
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), ClusterSpec(1, g, -(-total * 105 // (100 * g)), 1.0, 1.0))
    check(plan, seed=seed)


def test_programs_build_for_bench_configs():
    """C3 / C4 / C5 plans at G = 2, 4, 8: per-round pair counts match the
    schedule (asserted inside build_rank_program) and remap slices tile."""
    for g in (2, 4, 8):
        for batch in (W.c3_batch(g), W.c4_batch()):
            plan = P.build_plan(batch, W.cluster_for(batch, g))
            sched = S.build_schedule(plan)
            res = M.solve_remap(plan.tokens_per_rank, M.cost_matrix(W.cluster_for(batch, g)))
            total_pairs = 0
            for r in range(g):
                pr = build_rank_program(plan, sched, r, 32, res)
                total_pairs += pr.pairs_per_head()
                kept, (s0, s1), (r0, r1), send, recv = pr.remap.forward_slices(r)
                assert s1 - s0 == sum(send) and r1 - r0 == sum(recv)
            assert total_pairs == sum(S.causal_pairs(n) for _, n in batch.sequences)


GOLDEN_PERM = os.path.join(os.path.dirname(__file__), "golden", "remap_permutation.json")


def test_remap_permutation_golden():
    """R3 row rule pinned: for each case, the (src rank, src row) of every
    linear-layout row (run-length encoded) equals the committed fixture."""
    doc = json.load(open(GOLDEN_PERM))
    for case in doc["cases"]:
        lay = M.remap_layout(case["counts"])
        assert lay.matrix.tolist() == case["matrix"]
        for r, blocks in enumerate(case["blocks"]):
            assert [list(b) for b in lay.source_of_linear_rows(r)] == blocks
        src = OR.source_map(case["counts"], lay.matrix)
        for r, blocks in enumerate(case["blocks"]):
            want = np.concatenate([np.stack([np.full(n, s), np.arange(o, o + n)], 1) for s, o, n in blocks]) \
                if blocks else np.zeros((0, 2))
            assert np.array_equal(src[r], want)


# ------------------------------------------------------------------ backward work lists

def _causal_grads_f64(q, k, v, do, scale):
    """Whole-sequence causal attention gradients (numpy fp64), GQA by h // grp."""
    n, hq, d = q.shape
    grp = hq // k.shape[1]
    dq, dk, dv = np.zeros(q.shape), np.zeros(k.shape), np.zeros(k.shape)
    o = np.zeros(q.shape)
    lse = np.zeros((hq, n))
    mask = np.tril(np.ones((n, n), bool))
    for h in range(hq):
        s = q[:, h] @ k[:, h // grp].T * scale
        s = np.where(mask, s, -np.inf)
        m = s.max(1, keepdims=True)
        p = np.exp(s - m)
        l = p.sum(1, keepdims=True)
        p /= l
        o[:, h] = p @ v[:, h // grp]
        lse[h] = (m + np.log(l))[:, 0]
        dp = do[:, h] @ v[:, h // grp].T
        ds = p * (dp - (do[:, h] * o[:, h]).sum(1, keepdims=True))
        dq[:, h] = ds @ k[:, h // grp] * scale
        dk[:, h // grp] += ds.T @ q[:, h] * scale
        dv[:, h // grp] += p.T @ do[:, h]
    return o, lse, dq, dk, dv


def test_bwd_worklist_interpreter_matches_dense_gradients():
    """The backward work-item contract (64-row query blocks from the first
    visible one, grouped query segments) executed by the CPU interpreter
    reproduces dense causal gradients, and covers exactly the visible pairs."""
    from oracle.worklist import run_bwd_items
    from paper_2509_21841_b200.worklist import QueryFragment, build_bwd_worklist
    rng = np.random.default_rng(0)
    lens = [300, 70, 129]
    hq, hkv, d = 4, 2, 16
    t = sum(lens)
    q, k, v, do = (rng.standard_normal((t, h, d)) for h in (hq, hkv, hkv, hq))
    frags, r = [], 0
    for n in lens:
        frags.append(QueryFragment(row0=r, pos0=0, length=n, segs=[(r, 0, n)]))
        r += n
    wl = build_bwd_worklist(frags, hkv)
    assert wl.pairs_per_head == sum(n * (n + 1) // 2 for n in lens)
    scale = d ** -0.5
    ref = [np.zeros(x.shape) for x in (q, q, k, k)]
    o = np.zeros(q.shape)
    lse = np.zeros((hq, t))
    r = 0
    for n in lens:
        so, sl, sq_, sk_, sv_ = _causal_grads_f64(q[r:r + n], k[r:r + n], v[r:r + n], do[r:r + n], scale)
        o[r:r + n], lse[:, r:r + n] = so, sl
        ref[1][r:r + n], ref[2][r:r + n], ref[3][r:r + n] = sq_, sk_, sv_
        r += n
    delta = np.einsum("thd,thd->ht", do, o)
    dq, dk, dv, pairs = run_bwd_items(wl.items, wl.qsegs, q, k, v, do, lse, delta, scale)
    assert pairs == wl.pairs_per_head
    np.testing.assert_allclose(dq, ref[1], atol=1e-10)
    np.testing.assert_allclose(dk, ref[2], atol=1e-10)
    np.testing.assert_allclose(dv, ref[3], atol=1e-10)


@pytest.mark.parametrize("g", [2, 4, 8])
def test_bwd_program_covers_forward_pairs_with_disjoint_tiles(g):
    from paper_2509_21841_b200 import plan as P, schedule as S, workloads as W
    from paper_2509_21841_b200.program import build_bwd_program, build_rank_program
    b = W.c3_batch(g)
    plan = P.build_plan(b, W.cluster_for(b, g))
    sched = S.build_schedule(plan)
    for r in range(g):
        prog = build_rank_program(plan, sched, r, 32)
        bp = build_bwd_program(prog, 8)  # asserts pair counts against the forward lists
        for wl in [bp.local] + [w for lists in bp.rounds for w in lists]:
            tiles = set()
            for it in wl.items:
                key = (int(it["kv_head"]), int(it["kv_row0"]) // 128, int(it["kv_row0"]))
                assert key not in tiles
                tiles.add(key)
        for rp, up in zip(prog.rings, bp.unpack_ranges):
            assert np.array_equal(up[:, 0], rp.pack_ranges[:, 1]) and np.array_equal(up[:, 1], rp.pack_ranges[:, 0])


def _makespan(schedule, num_ranks, fill):
    """Cost-model makespan (pairs as time) of the ring list schedule with
    ``fill[r][j]`` local pairs run by rank r before its j-th ring and the rest
    after its last ring (reference simulator.py:136-187 ordering rules)."""
    in_ring = {s.sequence_id for rs in schedule.rings() for s in rs.ring.sequences}
    local = [0] * num_ranks
    for t in schedule.local_tasks:
        if t.sequence_id not in in_ring:
            local[t.rank] += t.compute_pairs
    t_now = [0] * num_ranks
    left = list(local)
    seen = [0] * num_ranks
    for rs in schedule.rings():
        members = rs.ring.members
        for m in members:
            take = fill[m][seen[m]]
            t_now[m] += take
            left[m] -= take
            seen[m] += 1
        start = max(t_now[m] for m in members)
        end = start + max(sum(rd.compute_pairs for rd in rs.rounds[i]) for i in range(len(members)))
        for m in members:
            t_now[m] = end
    return max(t + l for t, l in zip(t_now, left))


@pytest.mark.parametrize("seed", range(30))
def test_local_fill_never_lengthens_the_modelled_step(seed):
    """program.local_fill_plan (locals fill predicted ring waits) against
    "all locals first" under the same cost model: never longer, and every
    rank's local items are split into in-order chunks that cover the list."""
    from paper_2509_21841_b200.program import local_fill_plan
    rng = np.random.default_rng(seed)
    g = int(rng.choice([2, 3, 4, 5, 8]))
    lengths = [int(x) for x in rng.integers(1, 6000, size=int(rng.integers(3, 14)))]
    lengths.append(int(sum(lengths)))  # long enough to need a ring
    total = sum(lengths)
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), ClusterSpec(1, g, -(-total * 105 // (100 * g)),
                                                                              1.0, 1.0))
    sched = S.build_schedule(plan)
    fill = local_fill_plan(sched, g)
    in_ring = {s.sequence_id for rs in sched.rings() for s in rs.ring.sequences}
    local = [0] * g
    for t in sched.local_tasks:
        if t.sequence_id not in in_ring:
            local[t.rank] += t.compute_pairs
    first = {r: [local[r] if j == 0 else 0 for j in range(len(fill[r]))] for r in range(g)}
    assert _makespan(sched, g, fill) <= _makespan(sched, g, first)
    for r in range(g):
        prog = build_rank_program(plan, sched, r, 4)
        assert len(prog.local_cuts) == len(prog.rings)
        assert all(a <= b for a, b in zip(prog.local_cuts, prog.local_cuts[1:]))
        assert all(0 <= c <= prog.local.n_items and c % 2 == 0 for c in prog.local_cuts)
        assert sum(fill[r]) <= local[r]
