"""Pin the remap row rule (R3): tests/golden/remap_permutation.json.

Counts come from the reference's own plans (tokens_per_rank of the C1/C4/C5
plans, via the reference planner) and M from the reference solve_remap;
the blocks are the builder-defined row rule."""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from varlenplan import partitioner as rp, remapping as rr, topology as rt, workload as rw  # noqa: E402
from paper_2509_21841_b200 import workloads as W  # noqa: E402


def blocks_for(counts, m):
    d = len(counts)
    q, rem = divmod(sum(counts), d)
    b = [q + (i < rem) for i in range(d)]
    out = []
    for j in range(d):
        bl = [[j, 0, min(counts[j], b[j])]] if min(counts[j], b[j]) else []
        for s in range(d):
            if m[s][j]:
                bl.append([s, b[s] + sum(m[s][:j]), m[s][j]])
        out.append(bl)
    return out


cases = []
inv = 4096 / 900e9
todo = [("C1", [66, 73, 306, 41, 169, 241, 53, 37], (1, 2, 497, 1.0, 1.0))]
for g in (2, 4, 8):
    b = W.c4_batch()
    todo.append((f"C4-G{g}", [n for _, n in b.sequences], (1, g, -(-1050 * b.total_tokens // (1000 * g)), inv, inv)))
for name, lengths, args in todo:
    cl = rt.ClusterSpec(*args)
    plan = rp.build_plan(rw.SequenceBatch(tuple(enumerate(lengths))), cl)
    counts = list(plan.tokens_per_rank)
    m = rr.solve_remap(counts, rr.cost_matrix(cl)).matrix.tolist()
    cases.append({"name": name, "counts": counts, "matrix": m, "blocks": blocks_for(counts, m)})
for counts in ([262144, 0, 0, 0, 0, 0, 0, 0], [65536, 0, 65536, 0, 65536, 0, 65536, 0], [10, 0, 7, 3]):
    d = len(counts)
    cost = [[0.0 if i == j else 1.0 for j in range(d)] for i in range(d)]
    m = rr.solve_remap(counts, cost).matrix.tolist()
    cases.append({"name": f"stress-{counts[:3]}", "counts": counts, "matrix": m, "blocks": blocks_for(counts, m)})
json.dump({"generator": "tests/golden/make_remap_golden.py", "cases": cases},
          open(os.path.join(HERE, "remap_permutation.json"), "w"), indent=0)
print(len(cases), "cases")
