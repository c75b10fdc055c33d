"""The paper's comparison strategies as executable plans.

Restates the reference comparison planners (``baselines.py:51-202``) so the
same batch can be *run* on the GPUs under each strategy and the speed-up of
Zeppelin's plan measured instead of modelled:

* ``te_cp``     every sequence zigzag-split over ALL ranks in one global ring
                (Transformer-Engine context parallelism);
* ``llama_cp``  the same even layout, KV all-gathered before attention;
* ``hybrid_dp`` sequences longer than min(P*L*cp_fraction, L) ride the global
                ring, the rest are packed per rank by LPT on len^2 into
                capacity-bounded micro-batches.

Plans are bit-identical to the reference's (tests/test_planner_parity.py).
"""

from __future__ import annotations

from .cluster import ClusterSpec
from .plan import Fragment, InfeasibleBatch, PlacementPlan, first_over_capacity, validate_plan
from .schedule import (
    INTER_NODE,
    INTRA_NODE,
    LOCAL,
    RingGroup,
    RingSequence,
    balanced_zigzag_sizes,
    ranges_from_sizes,
)

STRATEGIES = ("zeppelin", "te_cp", "llama_cp", "hybrid_dp")


def _zone(ranks: set[int], cluster: ClusterSpec) -> str:
    if len({cluster.node_of(r) for r in ranks}) >= 2:
        return INTER_NODE
    return INTRA_NODE if len(ranks) >= 2 else LOCAL


def _buckets(fragments, cluster: ClusterSpec):
    out = []
    for node in range(cluster.num_nodes):
        acc: dict[int, int] = {}
        for r in cluster.ranks_of_node(node):
            for f in fragments[r]:
                acc[f.sequence_id] = acc.get(f.sequence_id, 0) + f.tokens
        out.append(sorted(acc.items()))
    return out


def _spread_over_all(seqs, n_ranks: int, cluster: ClusterSpec, fragments, zone_of) -> list[RingSequence]:
    """Zigzag every sequence over all ranks, leftovers to the lightest ranks."""
    running = [0] * n_ranks
    ring: list[RingSequence] = []
    for sid, length in seqs:
        ranges = ranges_from_sizes(balanced_zigzag_sizes(length, n_ranks, running)) if n_ranks > 1 \
            else [[(0, length)]]
        held = set()
        for pos, rs in enumerate(ranges):
            for a, b in rs:
                fragments[pos].append(Fragment(sid, a, b, pos))
                running[pos] += b - a
                held.add(pos)
        zone_of[sid] = _zone(held, cluster)
        if n_ranks > 1:
            ring.append(RingSequence(sequence_id=sid, ranges_by_position=tuple(tuple(r) for r in ranges)))
    return ring


def _finish(strategy, batch, cluster, fragments, zone_of, ring, mb_counts, meta) -> PlacementPlan:
    rings = ()
    if ring:
        rings = (RingGroup(kind=INTER_NODE if cluster.num_nodes > 1 else INTRA_NODE,
                           members=tuple(range(cluster.num_ranks)), sequences=tuple(ring)),)
    for frs in fragments:
        frs.sort(key=lambda f: (f.micro_batch, f.sequence_id, f.start))
    return PlacementPlan(
        strategy=strategy, num_nodes=cluster.num_nodes, gpus_per_node=cluster.gpus_per_node, s1=0,
        s0_per_node=[0] * cluster.num_nodes, zone_of=zone_of, sequence_lengths=batch.lengths,
        node_buckets=_buckets(fragments, cluster), fragments=fragments, ring_groups=rings,
        tokens_per_rank=[sum(f.tokens for f in frs) for frs in fragments], micro_batch_counts=mb_counts,
        meta=meta)


def _checked(plan: PlacementPlan, batch, cluster: ClusterSpec) -> PlacementPlan:
    over = first_over_capacity(plan, cluster)
    if over is not None:
        raise InfeasibleBatch(f"rank {over} exceeds token capacity under the even split")
    validate_plan(plan, batch, cluster)
    return plan


def _even(batch, cluster: ClusterSpec, strategy: str) -> PlacementPlan:
    cap = cluster.num_ranks * cluster.token_capacity
    if batch.total_tokens > cap:
        raise InfeasibleBatch(f"batch of {batch.total_tokens} tokens exceeds cluster capacity {cap}")
    n = cluster.num_ranks
    fragments: list[list[Fragment]] = [[] for _ in range(n)]
    zone_of: dict[int, str] = {}
    ring = _spread_over_all(sorted(batch.sequences), n, cluster, fragments, zone_of)
    return _finish(strategy, batch, cluster, fragments, zone_of, ring, [1] * n, {})


def plan_te_cp(batch, cluster: ClusterSpec) -> PlacementPlan:
    return _checked(_even(batch, cluster, "te_cp"), batch, cluster)


def plan_llama_cp(batch, cluster: ClusterSpec) -> PlacementPlan:
    return _checked(_even(batch, cluster, "llama_cp"), batch, cluster)


def plan_hybrid_dp(batch, cluster: ClusterSpec, cp_fraction: float = 1.0) -> PlacementPlan:
    if cp_fraction <= 0:
        raise ValueError("cp_fraction must be > 0")
    n = cluster.num_ranks
    cap = cluster.token_capacity
    threshold = min(cluster.gpus_per_node * cap * cp_fraction, cap)
    ordered = sorted(batch.sequences)
    cp = [(sid, ln) for sid, ln in ordered if ln > threshold]
    dp = [(sid, ln) for sid, ln in ordered if ln <= threshold]
    if sum(ln for _, ln in cp) > n * cap:
        raise InfeasibleBatch("ring-phase sequences exceed the cluster's token capacity")
    fragments: list[list[Fragment]] = [[] for _ in range(n)]
    zone_of: dict[int, str] = {}
    ring = _spread_over_all(cp, n, cluster, fragments, zone_of)
    # LPT on len^2, then capacity-bounded micro-batches per rank
    work = [0] * n
    mine: list[list[tuple[int, int]]] = [[] for _ in range(n)]
    for sid, ln in sorted(dp, key=lambda t: (-t[1], t[0])):
        r = min(range(n), key=lambda i: (work[i], i))
        work[r] += ln * ln
        mine[r].append((sid, ln))
    counts = [1] * n
    for r, seqs in enumerate(mine):
        mb, used = 1, 0
        for sid, ln in seqs:
            if used and used + ln > cap:
                mb, used = mb + 1, 0
            used += ln
            fragments[r].append(Fragment(sid, 0, ln, r, micro_batch=mb))
            zone_of[sid] = LOCAL
        counts[r] = mb
    plan = _finish("hybrid_dp", batch, cluster, fragments, zone_of, ring, counts,
                   {"cp_sequences": [sid for sid, _ in cp]})
    return _checked(plan, batch, cluster)


def plan_for(strategy: str, batch, cluster: ClusterSpec) -> PlacementPlan:
    from .plan import build_plan
    return {"zeppelin": build_plan, "te_cp": plan_te_cp, "llama_cp": plan_llama_cp,
            "hybrid_dp": plan_hybrid_dp}[strategy](batch, cluster)
