"""Live parity against the reference implementation (container only).

Imports /root/reference/pkg/src read-only and compares plan bytes, schedule
tuples, remap matrices / objectives, routes and sampler draws on thousands of
seeded instances — the reference's own property-test populations
(test_partitioner.py:177-191, test_acceptance.py:128-150, test_remapping.py:
73-87) plus the single-box configs of this repo.  Skipped where the
reference is absent (the GPU box); tests/test_golden.py covers that case.
"""
import os
import random
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")]

if os.path.isdir(REF):
    sys.path.insert(0, REF)
    from varlenplan import attention_engine as ra
    from varlenplan import partitioner as rp
    from varlenplan import remapping as rr
    from varlenplan import routing as rrt
    from varlenplan import topology as rt
    from varlenplan import workload as rw
    from varlenplan import baselines as rb

from paper_2509_21841_b200 import baselines as BL
from paper_2509_21841_b200 import batch as B
from paper_2509_21841_b200 import cluster as C
from paper_2509_21841_b200 import plan as P
from paper_2509_21841_b200 import remap as M
from paper_2509_21841_b200 import routing as RT
from paper_2509_21841_b200 import schedule as S


def sched_tuple(s):
    return ([(x.ring.kind, x.ring.members,
              [[(q.position, q.round_index, q.compute_pairs, q.comm_tokens) for q in pos] for pos in x.rounds])
             for x in s.rings()],
            [(t.rank, t.sequence_id, t.compute_pairs) for t in s.local_tasks])


def compare(seqs, args):
    rc, mc = rt.ClusterSpec(*args), C.ClusterSpec(*args)
    rb, mb = rw.SequenceBatch(tuple(seqs)), B.SequenceBatch(tuple(seqs))
    outcome = []
    for build, b, c in ((rp.build_plan, rb, rc), (P.build_plan, mb, mc)):
        try:
            outcome.append(build(b, c))
        except RuntimeError as exc:
            outcome.append((type(exc).__name__, str(exc)))
    ref, mine = outcome
    if isinstance(ref, tuple):
        assert ref == mine
        return None
    assert rp.plan_to_json(ref) == P.plan_to_json(mine)
    assert sched_tuple(ra.build_schedule(ref)) == sched_tuple(S.build_schedule(mine))
    a = rr.solve_remap(ref.tokens_per_rank, rr.cost_matrix(rc))
    b = M.solve_remap(mine.tokens_per_rank, M.cost_matrix(mc))
    assert np.array_equal(a.matrix, b.matrix) and a.objective == b.objective
    assert np.array_equal(a.row_costs, b.row_costs)
    def routes(rs):
        return {k: ([(s.kind, s.source_rank, s.dest_rank, s.tokens, s.scope) for s in v.steps],
                    v.x1, v.x2, v.dispatch_time, v.transfer_time, v.combine_time) for k, v in rs.items()}
    assert routes(rrt.route_schedule(ra.build_schedule(ref), ref, rc)) == \
        routes(RT.route_schedule(S.build_schedule(mine), mine, mc))
    return mine


def test_random_small_clusters():
    rng = random.Random(99)
    done = 0
    for _ in range(1500):
        n, p, cap = rng.choice([1, 2, 3]), rng.choice([1, 2, 4, 8]), rng.randint(4, 40)
        lengths = [rng.randint(1, n * p * cap) for _ in range(rng.randint(0, 6))]
        if sum(lengths) > n * p * cap:
            continue
        compare(list(enumerate(lengths)), (n, p, cap, 1.0, 2.0))
        done += 1
    assert done > 300


def test_cluster_a_acceptance_population():
    ca, _ = rt.cluster_a()
    args = (ca.num_nodes, ca.gpus_per_node, ca.token_capacity, ca.inv_bw_intra, ca.inv_bw_inter, ca.nics_per_node)
    for name in ("arxiv", "github", "prolong64k"):
        for seed in range(200):
            rb = rw.sample_batch(rw.preset(name), 65536, seed)
            assert B.sample_batch(B.preset(name), 65536, seed).sequences == rb.sequences
            compare(list(rb.sequences), args)


@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_single_box_long_batches(g):
    inv = 4096 / 900e9
    for total in (65536, 262144, 524288):
        for name in ("arxiv", "github", "prolong64k"):
            for seed in range(8):
                seqs = list(rw.sample_batch(rw.preset(name), total, seed).sequences)
                compare(seqs, (1, g, -(-1050 * total // (1000 * g)), inv, inv))


def test_remap_random_instances():
    rng = random.Random(7)
    for _ in range(300):
        d = rng.randint(1, 8)
        counts = [rng.randint(0, 80) for _ in range(d)]
        if d % 2 == 0 and rng.random() < 0.5:
            cost = rr.cost_matrix(rt.ClusterSpec(2, d // 2, 1000, 1.0, rng.uniform(1.0, 20.0)))
        else:
            cost = np.full((d, d), rng.uniform(0.1, 5.0))
            np.fill_diagonal(cost, 0.0)
        a, b = rr.solve_remap(counts, cost), M.solve_remap(counts, cost)
        assert np.array_equal(a.matrix, b.matrix) and a.objective == b.objective
        if d > 1 and np.all(cost[~np.eye(d, dtype=bool)] == cost[0, 1]):
            assert np.array_equal(M.northwest_corner(counts), a.matrix)


def test_zigzag_helpers_and_pairs():
    rng = random.Random(4)
    for _ in range(500):
        g = rng.randint(1, 16)
        s = rng.randint(1, 600)
        loads = [rng.randint(0, 50) for _ in range(g)]
        assert ra.balanced_zigzag_sizes(s, g, loads) == S.balanced_zigzag_sizes(s, g, loads)
        assert ra.zigzag_ranges_by_position(s, g) == S.zigzag_ranges_by_position(s, g)
        assert ra.split_even(s, g) == S.split_even(s, g)
        a = rng.randint(0, 300)
        q = (a, a + rng.randint(0, 100))
        kv = []
        at = 0
        for _ in range(rng.randint(0, 3)):
            lo = at + rng.randint(0, 40)
            kv.append((lo, lo + rng.randint(0, 60)))
            at = kv[-1][1]
        assert ra.visible_pairs(q, kv) == S.visible_pairs(q, kv)


def test_intermediate_levels_match():
    """partition_inter_node / partition_intra_node results, field by field."""
    rng = random.Random(5)
    for _ in range(300):
        n, p, cap = rng.choice([1, 2, 3]), rng.choice([1, 2, 4]), rng.randint(4, 40)
        lengths = [rng.randint(1, n * p * cap // 2 + 1) for _ in range(rng.randint(1, 6))]
        if sum(lengths) > n * p * cap:
            continue
        args = (n, p, cap, 1.0, 2.0)
        rb, mb = rw.SequenceBatch(tuple(enumerate(lengths))), B.SequenceBatch(tuple(enumerate(lengths)))
        try:
            a = rp.partition_inter_node(rb, rt.ClusterSpec(*args))
        except rp.InfeasibleBatch:
            with pytest.raises(P.InfeasibleBatch):
                P.partition_inter_node(mb, C.ClusterSpec(*args))
            continue
        b = P.partition_inter_node(mb, C.ClusterSpec(*args))
        assert (a.s1, a.restarts) == (b.s1, b.restarts)
        for x, y in zip(a.buckets, b.buckets):
            assert [(c.sequence_id, c.start, c.end) for c in x.chunks] == [(c.sequence_id, c.start, c.end) for c in y.chunks]
            assert x.own == y.own
            try:
                ia = rp.partition_intra_node(x, rt.ClusterSpec(*args))
            except rp.InfeasibleNode:
                with pytest.raises(P.InfeasibleNode):
                    P.partition_intra_node(y, C.ClusterSpec(*args))
                continue
            ib = P.partition_intra_node(y, C.ClusterSpec(*args))
            assert (ia.s0, ia.restarts) == (ib.s0, ib.restarts)
            assert [[(e.sequence_id, e.start, e.end, e.kind) for e in d] for d in ia.devices] == \
                   [[(e.sequence_id, e.start, e.end, e.kind) for e in d] for d in ib.devices]


@pytest.mark.parametrize("strategy", ["te_cp", "llama_cp", "hybrid_dp"])
def test_baseline_planners_bit_exact(strategy):
    rng = random.Random(17)
    fn_ref = {"te_cp": rb.plan_te_cp, "llama_cp": rb.plan_llama_cp, "hybrid_dp": rb.plan_hybrid_dp}[strategy]
    fn_me = {"te_cp": BL.plan_te_cp, "llama_cp": BL.plan_llama_cp, "hybrid_dp": BL.plan_hybrid_dp}[strategy]
    cases = []
    for _ in range(300):
        n, p, cap = rng.choice([1, 2]), rng.choice([1, 2, 4, 8]), rng.randint(4, 60)
        cases.append(([rng.randint(1, n * p * cap // 2 + 1) for _ in range(rng.randint(1, 7))], (n, p, cap, 1.0, 2.0)))
    inv = 4096 / 900e9
    for g in (2, 4, 8):
        for name in ("arxiv", "github", "prolong64k"):
            for seed in range(3):
                seqs = rw.sample_batch(rw.preset(name), 262144, seed).sequences
                cases.append(([n for _, n in seqs], (1, g, -(-1050 * 262144 // (1000 * g)), inv, inv)))
    for lengths, args in cases:
        rb_, mb_ = rw.SequenceBatch(tuple(enumerate(lengths))), B.SequenceBatch(tuple(enumerate(lengths)))
        try:
            a = fn_ref(rb_, rt.ClusterSpec(*args))
        except Exception as exc:
            with pytest.raises(Exception) as info:
                fn_me(mb_, C.ClusterSpec(*args))
            assert (type(info.value).__name__, str(info.value)) == (type(exc).__name__, str(exc))
            continue
        b = fn_me(mb_, C.ClusterSpec(*args))
        assert rp.plan_to_json(a) == P.plan_to_json(b)
        assert sched_tuple(ra.build_schedule(a)) == sched_tuple(S.build_schedule(b))
