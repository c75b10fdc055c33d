"""Generate tests/golden/planner_golden.json from the REFERENCE implementation.

Run in the container that has /root/reference (read-only):
    python tests/golden/make_golden.py
The fixture pins, for every case, the reference's plan (sha256 of
plan_to_json), ring/local schedule (sha256 of its tuple form), tokens per rank
and remap matrix + objective.  tests/test_golden.py checks this repo's
planner against it on any host (the GPU box has no /root/reference).
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from varlenplan import attention_engine as ra  # noqa: E402
from varlenplan import partitioner as rp  # noqa: E402
from varlenplan import remapping as rr  # noqa: E402
from varlenplan import topology as rt  # noqa: E402
from varlenplan import workload as rw  # noqa: E402

from paper_2509_21841_b200 import workloads as W  # noqa: E402  (batch shapes only)


def schedule_tuple(s):
    return (
        [(x.ring.kind, list(x.ring.members),
          [[(q.position, q.round_index, q.compute_pairs, q.comm_tokens) for q in pos] for pos in x.rounds])
         for x in s.rings()],
        [(t.rank, t.sequence_id, t.compute_pairs) for t in s.local_tasks],
    )


def sha(obj) -> str:
    text = obj if isinstance(obj, str) else json.dumps(obj, sort_keys=True)
    return hashlib.sha256(text.encode()).hexdigest()


def case(name, lengths, cluster_args, keep_json=False):
    cl = rt.ClusterSpec(*cluster_args)
    batch = rw.SequenceBatch(tuple(enumerate(lengths)) if not isinstance(lengths[0], (list, tuple))
                             else tuple(tuple(x) for x in lengths))
    out = {"name": name, "cluster": list(cluster_args), "sequences": [list(x) for x in batch.sequences]}
    try:
        plan = rp.build_plan(batch, cl)
    except rp.InfeasibleBatch as exc:
        out["error"] = [type(exc).__name__, str(exc)]
        return out
    text = rp.plan_to_json(plan)
    out["plan_sha256"] = sha(text)
    if keep_json:
        out["plan_json"] = text
    sched = ra.build_schedule(plan)
    out["schedule_sha256"] = sha(schedule_tuple(sched))
    out["ring_pairs"] = sum(q.compute_pairs for x in sched.rings() for pos in x.rounds for q in pos)
    out["local_pairs"] = sum(t.compute_pairs for t in sched.local_tasks)
    out["tokens_per_rank"] = list(plan.tokens_per_rank)
    res = rr.solve_remap(plan.tokens_per_rank, rr.cost_matrix(cl))
    out["remap_matrix"] = res.matrix.tolist()
    out["remap_objective"] = res.objective
    return out


def main():
    cases = []
    # C1 golden
    cases.append(case("C1", [66, 73, 306, 41, 169, 241, 53, 37], (1, 2, 497, 1.0, 1.0), keep_json=True))
    inv = 4096 / 900e9
    # C2: 64K presets x seeds, one B200
    for p in ("arxiv", "github", "prolong64k"):
        for seed in range(5):
            b = rw.sample_batch(rw.preset(p), 65536, seed)
            cases.append(case(f"C2-{p}-{seed}", list(b.sequences), (1, 1, 68813, inv, inv)))
    # C3 / C4 / C5 batch shapes at G = 2/4/8 (single NVSwitch box, 5% slack)
    for g in (2, 4, 8):
        b3 = W.c3_batch(g)
        cap3 = -(-1050 * b3.total_tokens // (1000 * g))
        cases.append(case(f"C3-G{g}", [list(x) for x in b3.sequences], (1, g, cap3, inv, inv), keep_json=True))
        b4 = W.c4_batch()
        cap4 = -(-1050 * b4.total_tokens // (1000 * g))
        cases.append(case(f"C4-G{g}", [list(x) for x in b4.sequences], (1, g, cap4, inv, inv), keep_json=True))
    # single-box presets at 64K / 256K, G = 2/4/8
    for g in (2, 4, 8):
        for total in (65536, 262144):
            for p in ("arxiv", "github", "prolong64k"):
                for seed in range(4):
                    b = rw.sample_batch(rw.preset(p), total, seed)
                    cap = -(-1050 * total // (1000 * g))
                    cases.append(case(f"box-G{g}-{total}-{p}-{seed}", list(b.sequences), (1, g, cap, inv, inv)))
    # two-node cluster_a (inter-node rings, non-uniform remap costs)
    ca, _ = rt.cluster_a()
    ca_args = (ca.num_nodes, ca.gpus_per_node, ca.token_capacity, ca.inv_bw_intra, ca.inv_bw_inter, ca.nics_per_node)
    for p in ("arxiv", "github", "prolong64k"):
        for seed in range(10):
            b = rw.sample_batch(rw.preset(p), 65536, seed)
            cases.append(case(f"cluster_a-{p}-{seed}", list(b.sequences), ca_args))
    # random small clusters (feasible and infeasible)
    rng = random.Random(2024)
    for i in range(150):
        n = rng.choice([1, 2, 3])
        p = rng.choice([1, 2, 4, 8])
        cap = rng.randint(4, 60)
        lengths = [rng.randint(1, max(1, n * p * cap // 2)) for _ in range(rng.randint(1, 7))]
        cases.append(case(f"small-{i}", lengths, (n, p, cap, 1.0, 2.0)))
    # remap-only instances (uniform and two-node costs)
    remaps = []
    rng = random.Random(7)
    for i in range(120):
        d = rng.choice([2, 3, 4, 6, 8])
        counts = [rng.randint(0, 60) for _ in range(d)]
        if d % 2 == 0 and rng.random() < 0.5:
            cl = rt.ClusterSpec(2, d // 2, 1000, 1.0, rng.uniform(1.0, 20.0))
            cost = rr.cost_matrix(cl)
        else:
            cost = [[0.0 if a == b else 1.5 for b in range(d)] for a in range(d)]
        res = rr.solve_remap(counts, cost)
        remaps.append({"counts": counts, "cost": [list(map(float, r)) for r in cost],
                       "matrix": res.matrix.tolist(), "objective": res.objective,
                       "target": rr.target_distribution(counts)})
    # sampler draws
    samples = []
    for p in ("arxiv", "github", "prolong64k"):
        for seed in range(3):
            samples.append({"preset": p, "total": 65536, "seed": seed,
                            "sequences": [list(x) for x in rw.sample_batch(rw.preset(p), 65536, seed).sequences]})
    doc = {"generator": "tests/golden/make_golden.py (reference varlenplan 0.1.0 from /root/reference/pkg/src)",
           "cases": cases, "remaps": remaps, "samples": samples}
    path = os.path.join(HERE, "planner_golden.json")
    with open(path, "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print(f"wrote {path}: {len(cases)} plan cases, {len(remaps)} remap cases, {len(samples)} samples")


if __name__ == "__main__":
    main()
