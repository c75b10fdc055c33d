"""Planner / schedule / remap-matrix parity against committed reference fixtures.

tests/golden/planner_golden.json was produced by tests/golden/make_golden.py
from the reference implementation itself; this test runs on any host (the GPU
box has no /root/reference) and requires bit-exact agreement.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2509_21841_b200 import batch as B
from paper_2509_21841_b200 import cluster as C
from paper_2509_21841_b200 import plan as P
from paper_2509_21841_b200 import remap as M
from paper_2509_21841_b200 import schedule as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "planner_golden.json")))


def _sha(obj):
    text = obj if isinstance(obj, str) else json.dumps(obj, sort_keys=True)
    return hashlib.sha256(text.encode()).hexdigest()


def schedule_tuple(s):
    return (
        [(x.ring.kind, list(x.ring.members),
          [[(q.position, q.round_index, q.compute_pairs, q.comm_tokens) for q in pos] for pos in x.rounds])
         for x in s.rings()],
        [(t.rank, t.sequence_id, t.compute_pairs) for t in s.local_tasks],
    )


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=[c["name"] for c in GOLDEN["cases"]])
def test_plan_schedule_remap_bit_exact(case):
    cluster = C.ClusterSpec(*case["cluster"])
    batch = B.SequenceBatch(tuple(tuple(x) for x in case["sequences"]))
    if "error" in case:
        with pytest.raises(P.InfeasibleBatch) as info:
            P.build_plan(batch, cluster)
        assert [type(info.value).__name__, str(info.value)] == case["error"]
        return
    plan = P.build_plan(batch, cluster)
    text = P.plan_to_json(plan)
    if "plan_json" in case:
        assert text == case["plan_json"]
    assert _sha(text) == case["plan_sha256"]
    sched = S.build_schedule(plan)
    assert _sha(schedule_tuple(sched)) == case["schedule_sha256"]
    assert plan.tokens_per_rank == case["tokens_per_rank"]
    res = M.solve_remap(plan.tokens_per_rank, M.cost_matrix(cluster))
    assert res.matrix.tolist() == case["remap_matrix"]
    assert res.objective == case["remap_objective"]
    # plan JSON round trip
    again = P.plan_from_json(text)
    assert again.fragments == plan.fragments and again.ring_groups == plan.ring_groups


@pytest.mark.parametrize("idx", range(len(GOLDEN["remaps"])))
def test_remap_matrix_bit_exact(idx):
    r = GOLDEN["remaps"][idx]
    res = M.solve_remap(r["counts"], np.array(r["cost"]))
    assert res.matrix.tolist() == r["matrix"]
    assert res.objective == r["objective"]
    assert M.target_distribution(r["counts"]) == r["target"]


def test_uniform_cost_matrix_is_northwest_corner():
    for r in GOLDEN["remaps"]:
        cost = np.array(r["cost"])
        off = cost[~np.eye(len(cost), dtype=bool)]
        if off.size and np.all(off == off[0]):
            assert M.northwest_corner(r["counts"]).tolist() == r["matrix"]


@pytest.mark.parametrize("s", GOLDEN["samples"], ids=lambda s: f"{s['preset']}-{s['seed']}")
def test_sampler_draws_identical(s):
    got = B.sample_batch(B.preset(s["preset"]), s["total"], s["seed"])
    assert [list(x) for x in got.sequences] == s["sequences"]


def test_c1_appendix_b():
    """SURVEY Appendix B golden example, field by field."""
    from paper_2509_21841_b200 import workloads as W
    plan = P.build_plan(W.c1_batch(), W.c1_cluster())
    assert hashlib.sha256(P.plan_to_json(plan).encode()).hexdigest()[:16] == "777c1f7088f04e67"
    assert [(f.sequence_id, f.start, f.end) for f in plan.fragments[0]] == [
        (0, 0, 66), (2, 0, 77), (2, 230, 306), (5, 0, 241), (7, 0, 37)]
    assert [(f.sequence_id, f.start, f.end) for f in plan.fragments[1]] == [
        (1, 0, 73), (2, 77, 154), (2, 154, 230), (3, 0, 41), (4, 0, 169), (6, 0, 53)]
    sched = S.build_schedule(plan)
    rounds = [[(q.round_index, q.compute_pairs, q.comm_tokens) for q in pos] for pos in sched.rings()[0].rounds]
    assert rounds == [[(0, 11781, 153), (1, 11628, 153)], [(0, 11781, 153), (1, 11781, 153)]]
    assert [(t.rank, t.sequence_id, t.compute_pairs) for t in sched.local_tasks] == [
        (0, 0, 2211), (0, 5, 29161), (0, 7, 703), (1, 1, 2701), (1, 3, 861), (1, 4, 14365), (1, 6, 1431)]
    res = M.solve_remap(plan.tokens_per_rank, M.cost_matrix(W.c1_cluster()))
    assert M.target_distribution(plan.tokens_per_rank) == [493, 493]
    assert res.matrix.tolist() == [[0, 4], [0, 0]]
    assert res.objective == 3.9999999962747097
