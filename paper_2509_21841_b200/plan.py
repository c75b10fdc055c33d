"""Hierarchical sequence partitioner (paper Alg. 1 + 2) — host planner.

Restates the reference partitioner (``partitioner.py``) so that, for the same
``SequenceBatch`` and ``ClusterSpec``, ``plan_to_json(build_plan(...))`` is
byte-identical to the reference's.  Parity is enforced by
``tests/test_planner_parity.py`` (live reference, in this container) and
``tests/golden/plans.json`` (committed fixtures, everywhere).

Structure (reference line numbers in brackets):
  level 1  ``partition_inter_node``  [169-287]  node buckets; sequences with
           length >= s1 are cut into k = ceil(len*N / sum_z2) chunks on
           distinct least-loaded nodes, the rest go whole to the least-loaded
           node; an overflow lowers s1 to the longest whole sequence and
           restarts; a chunk that fits nowhere re-splits the sequence holding
           the largest chunks [154-166].
  level 2  ``partition_intra_node``  [290-410]  per node; chunks are spread
           evenly over all devices, sequences >= s0 are split into
           k = ceil(len^2*P / sum_z1 len^2) fragments placed round-robin from
           a cursor, the rest go whole to the least-loaded device.
  compose  ``build_plan``  [413-513]  capacity reconciliation loop.
  layout   ``_assemble``  [516-648]  ring jobs, zigzag fragments, zones.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

from .cluster import ClusterSpec
from .schedule import (
    INTER_NODE,
    INTRA_NODE,
    LOCAL,
    RingGroup,
    RingSequence,
    balanced_zigzag_sizes,
    contiguous_ranges,
    ranges_from_sizes,
    split_even,
)


class InfeasibleBatch(RuntimeError):
    """The batch cannot be placed within the cluster's token capacity."""


class InfeasibleNode(InfeasibleBatch):
    """A node bucket cannot be spread over its devices within capacity."""


class PlanValidationError(RuntimeError):
    """A plan failed its internal consistency check (bug guard)."""


@dataclass(frozen=True)
class Fragment:
    sequence_id: int
    start: int
    end: int
    rank: int
    micro_batch: int = 0

    @property
    def tokens(self) -> int:
        return self.end - self.start


@dataclass(frozen=True)
class NodeChunk:
    sequence_id: int
    start: int
    end: int

    @property
    def tokens(self) -> int:
        return self.end - self.start


@dataclass
class NodeBucket:
    chunks: list[NodeChunk] = field(default_factory=list)
    own: list[tuple[int, int]] = field(default_factory=list)

    @property
    def tokens(self) -> int:
        return sum(c.tokens for c in self.chunks) + sum(n for _, n in self.own)


@dataclass
class InterNodeAssignment:
    buckets: list[NodeBucket]
    s1: int
    restarts: int


@dataclass(frozen=True)
class DeviceEntry:
    sequence_id: int
    start: int
    end: int
    kind: str  # "chunk_part" | "split" | "whole"

    @property
    def tokens(self) -> int:
        return self.end - self.start


@dataclass
class IntraNodeAssignment:
    devices: list[list[DeviceEntry]]
    s0: int
    restarts: int


@dataclass
class PlacementPlan:
    strategy: str
    num_nodes: int
    gpus_per_node: int
    s1: int
    s0_per_node: list[int]
    zone_of: dict[int, str]
    sequence_lengths: dict[int, int]
    node_buckets: list[list[tuple[int, int]]]
    fragments: list[list[Fragment]]
    ring_groups: tuple[RingGroup, ...]
    tokens_per_rank: list[int]
    micro_batch_counts: list[int]
    meta: dict

    @property
    def num_ranks(self) -> int:
        return self.num_nodes * self.gpus_per_node

    @property
    def device_buckets(self) -> list[list[Fragment]]:
        return self.fragments

    def total_tokens(self) -> int:
        return sum(self.tokens_per_rank)


# ----------------------------------------------------------------- helpers

def _longest_first(pairs) -> list[tuple[int, int]]:
    return sorted(pairs, key=lambda sl: (-sl[1], sl[0]))


def _argmin_load(loads: list[int]) -> int:
    return min(range(len(loads)), key=lambda i: (loads[i], i))


class _SplitFailure(Exception):
    """A sequence found no fitting placement; ``placed`` holds (len, k) of the
    sequences already placed in this pass, the candidates for a re-split."""

    def __init__(self, sid: int, length: int, placed: dict[int, tuple[int, int]]):
        super().__init__(f"sequence {sid} ({length} tokens) does not fit")
        self.sid = sid
        self.placed = placed


def _resplit_heaviest(fail: _SplitFailure, overrides: dict[int, int], max_parts: int) -> bool:
    """Give one more part to the placed sequence with the largest parts
    (ties: lowest id).  False when every candidate is fully split."""
    best = None
    for sid, (length, k) in fail.placed.items():
        if k >= max_parts:
            continue
        key = (length / k, -sid)
        if best is None or key > best[0]:
            best = (key, sid, k)
    if best is None:
        return False
    overrides[best[1]] = best[2] + 1
    return True


def _try_parts(length: int, k_first: int, n_bins: int, loads: list[int], cap: int, pick):
    """Shared retry loop of both levels: for k = min(k_first, n)..n split the
    sequence evenly into k parts and ask ``pick(sizes, trial_loads)`` for a
    bin per part; first success wins.  Returns (k, sizes, bins) or None."""
    for k in range(min(k_first, n_bins), n_bins + 1):
        sizes = split_even(length, k)
        bins = pick(sizes, list(loads))
        if bins is not None:
            return k, sizes, bins
    return None


# ----------------------------------------------------------------- level 1

def _pick_least_loaded(loads: list[int], cap: int):
    def pick(sizes, trial):
        order = sorted(range(len(loads)), key=lambda i: (loads[i], i))  # pre-placement loads
        chosen: list[int] = []
        for size in sizes:
            hit = next((i for i in order if i not in chosen and trial[i] + size <= cap), None)
            if hit is None:
                return None
            chosen.append(hit)
            trial[hit] += size
        return chosen
    return pick


def _inter_pass(order, n_nodes: int, node_cap: int, overrides: dict[int, int]) -> InterNodeAssignment:
    s1 = node_cap
    restarts = 0
    while True:
        buckets = [NodeBucket() for _ in range(n_nodes)]
        loads = [0] * n_nodes
        chunked = [(sid, n) for sid, n in order if n >= s1]
        whole = [(sid, n) for sid, n in order if n < s1]
        chunked_total = sum(n for _, n in chunked)
        placed: dict[int, tuple[int, int]] = {}
        for sid, n in chunked:
            k0 = max(1, -(-n * n_nodes // chunked_total), overrides.get(sid, 1))
            hit = _try_parts(n, k0, n_nodes, loads, node_cap, _pick_least_loaded(loads, node_cap))
            if hit is None:
                raise _SplitFailure(sid, n, placed)
            k, sizes, bins = hit
            for (a, b), node in zip(contiguous_ranges(sizes), bins):
                if b > a:
                    buckets[node].chunks.append(NodeChunk(sid, a, b))
                    loads[node] += b - a
            placed[sid] = (n, k)
        overflow = False
        for sid, n in whole:
            node = _argmin_load(loads)
            if loads[node] + n > node_cap:
                s1 = max(m for _, m in whole)
                restarts += 1
                overflow = True
                break
            buckets[node].own.append((sid, n))
            loads[node] += n
        if not overflow:
            return InterNodeAssignment(buckets=buckets, s1=s1, restarts=restarts)
        if restarts > len(order) + 1:
            raise InfeasibleBatch("node threshold refinement did not converge")


def partition_inter_node(batch, cluster: ClusterSpec,
                         chunk_overrides: dict[int, int] | None = None) -> InterNodeAssignment:
    overrides = dict(chunk_overrides or {})
    n_nodes = cluster.num_nodes
    node_cap = cluster.gpus_per_node * cluster.token_capacity
    order = _longest_first(batch.sequences)
    total = sum(n for _, n in order)
    if total > n_nodes * node_cap:
        raise InfeasibleBatch(f"batch of {total} tokens exceeds cluster capacity {n_nodes * node_cap}")
    retries = (len(order) + 1) * n_nodes
    while True:
        try:
            return _inter_pass(order, n_nodes, node_cap, overrides)
        except _SplitFailure as fail:
            retries -= 1
            if retries < 0 or not _resplit_heaviest(fail, overrides, n_nodes):
                raise InfeasibleBatch(f"sequence {fail.sid} cannot be chunked across nodes") from None


# ----------------------------------------------------------------- level 2

def _pick_round_robin(cursor: int, cap: int):
    def pick(sizes, trial):
        p = len(trial)
        chosen: list[int] = []
        at = cursor
        for size in sizes:
            hit = None
            for step in range(p):
                dev = (at + step) % p
                if dev not in chosen and trial[dev] + size <= cap:
                    hit = dev
                    break
            if hit is None:
                return None
            chosen.append(hit)
            trial[hit] += size
            at = (hit + 1) % p
        return chosen
    return pick


def _intra_pass(node: NodeBucket, own, p: int, cap: int, overrides: dict[int, int]) -> IntraNodeAssignment:
    s0 = cap
    restarts = 0
    while True:
        devices: list[list[DeviceEntry]] = [[] for _ in range(p)]
        loads = [0] * p
        for chunk in node.chunks:
            spans = contiguous_ranges(split_even(chunk.tokens, p), offset=chunk.start)
            for dev, (a, b) in enumerate(spans):
                if b > a:
                    devices[dev].append(DeviceEntry(chunk.sequence_id, a, b, "chunk_part"))
                    loads[dev] += b - a
        split = [(sid, n) for sid, n in own if n >= s0]
        whole = [(sid, n) for sid, n in own if n < s0]
        sq_total = sum(n * n for _, n in split)
        cursor = 0
        placed: dict[int, tuple[int, int]] = {}
        for sid, n in split:
            k0 = max(1, -(-n * n * p // sq_total), overrides.get(sid, 1))
            hit = _try_parts(n, k0, p, loads, cap, _pick_round_robin(cursor, cap))
            if hit is None:
                raise _SplitFailure(sid, n, placed)
            k, sizes, bins = hit
            for (a, b), dev in zip(contiguous_ranges(sizes), bins):
                if b > a:
                    devices[dev].append(DeviceEntry(sid, a, b, "split"))
                    loads[dev] += b - a
            cursor = (bins[-1] + 1) % p
            placed[sid] = (n, k)
        overflow = False
        for sid, n in whole:
            dev = _argmin_load(loads)
            if loads[dev] + n > cap:
                s0 = max(m for _, m in whole)
                restarts += 1
                overflow = True
                break
            devices[dev].append(DeviceEntry(sid, 0, n, "whole"))
            loads[dev] += n
        if not overflow:
            return IntraNodeAssignment(devices=devices, s0=s0, restarts=restarts)
        if restarts > len(own) + 1:
            raise InfeasibleNode("device threshold refinement did not converge")


def partition_intra_node(node: NodeBucket, cluster: ClusterSpec,
                         split_overrides: dict[int, int] | None = None) -> IntraNodeAssignment:
    overrides = dict(split_overrides or {})
    p = cluster.gpus_per_node
    own = _longest_first(node.own)
    retries = (len(own) + 1) * p
    while True:
        try:
            return _intra_pass(node, own, p, cluster.token_capacity, overrides)
        except _SplitFailure as fail:
            retries -= 1
            if retries < 0 or not _resplit_heaviest(fail, overrides, p):
                raise InfeasibleNode(f"sequence {fail.sid} cannot be split within the node") from None


# ----------------------------------------------------------------- compose

def _chunk_counts(inter: InterNodeAssignment) -> dict[int, int]:
    counts: dict[int, int] = {}
    for bucket in inter.buckets:
        for c in bucket.chunks:
            counts[c.sequence_id] = counts.get(c.sequence_id, 0) + 1
    return counts


def _phase_load_exceeds(plan: PlacementPlan, rank: int, cap: int) -> bool:
    per_phase: dict[int, int] = {}
    for f in plan.fragments[rank]:
        per_phase[f.micro_batch] = per_phase.get(f.micro_batch, 0) + f.tokens
    return any(v > cap for v in per_phase.values())


def first_over_capacity(plan: PlacementPlan, cluster: ClusterSpec) -> int | None:
    for rank in range(plan.num_ranks):
        if _phase_load_exceeds(plan, rank, cluster.token_capacity):
            return rank
    return None


def _relieve_rank(plan: PlacementPlan, cluster: ClusterSpec, rank: int, inter: InterNodeAssignment,
                  node_overrides: dict[int, int], split_overrides: list[dict[int, int]]) -> bool:
    """Spread the heaviest non-local sequence of an over-capacity rank over
    one more node (if it is chunked across nodes) or one more device."""
    node = rank // cluster.gpus_per_node
    counts = _chunk_counts(inter)
    mine: dict[int, int] = {}
    for f in plan.fragments[rank]:
        mine[f.sequence_id] = mine.get(f.sequence_id, 0) + f.tokens
    candidates = sorted(((tok, sid) for sid, tok in mine.items() if plan.zone_of[sid] != LOCAL),
                        reverse=True)
    for _, sid in candidates:
        if plan.zone_of[sid] == INTER_NODE or sid in counts:
            current = max(counts.get(sid, 1), node_overrides.get(sid, 1))
            if current < cluster.num_nodes:
                node_overrides[sid] = current + 1
                return True
        else:
            spans = len({f.rank for frs in plan.fragments for f in frs if f.sequence_id == sid})
            current = max(spans, split_overrides[node].get(sid, 1))
            if current < cluster.gpus_per_node:
                split_overrides[node][sid] = current + 1
                return True
    return False


def build_plan(batch, cluster: ClusterSpec) -> PlacementPlan:
    node_overrides: dict[int, int] = {}
    split_overrides: list[dict[int, int]] = [{} for _ in range(cluster.num_nodes)]
    for attempt in range(cluster.num_ranks + 1):
        inter = partition_inter_node(batch, cluster, node_overrides)
        intra: list[IntraNodeAssignment] = []
        failed = None
        for n, bucket in enumerate(inter.buckets):
            try:
                intra.append(partition_intra_node(bucket, cluster, split_overrides[n]))
            except InfeasibleNode:
                failed = n
                break
        if failed is not None:
            # spread one of the failed node's chunked sequences over one more
            # node and redo level 1 (largest chunk first, then largest id)
            counts = _chunk_counts(inter)
            options = sorted(
                ((c.tokens, c.sequence_id) for c in inter.buckets[failed].chunks
                 if max(counts[c.sequence_id], node_overrides.get(c.sequence_id, 1)) < cluster.num_nodes),
                reverse=True)
            if not options:
                raise InfeasibleBatch(f"node {failed} cannot spread its bucket over its devices")
            sid = options[0][1]
            node_overrides[sid] = max(counts[sid], node_overrides.get(sid, 1)) + 1
            continue
        plan = _assemble(batch, cluster, inter, intra, attempt)
        over = first_over_capacity(plan, cluster)
        if over is None:
            validate_plan(plan, batch, cluster)
            return plan
        if not _relieve_rank(plan, cluster, over, inter, node_overrides, split_overrides):
            raise InfeasibleBatch("no split sequence available to relieve an over-capacity rank")
    raise InfeasibleBatch("capacity reconciliation exceeded its retry budget")


# ----------------------------------------------------------------- layout

class _Layout:
    """Mutable state while fragments are laid out: per-rank fragment lists,
    running token loads, zone labels and ring membership."""

    def __init__(self, cluster: ClusterSpec):
        self.p = cluster.gpus_per_node
        self.fragments: list[list[Fragment]] = [[] for _ in range(cluster.num_ranks)]
        self.zone_of: dict[int, str] = {}
        self.rings: dict[tuple[str, tuple[int, ...]], list[RingSequence]] = {}
        self.running: list[int] | None = None

    def place_whole(self, sid: int, length: int, rank: int) -> None:
        self.zone_of[sid] = LOCAL
        self.fragments[rank].append(Fragment(sid, 0, length, rank))
        if self.running is not None:
            self.running[rank] += length

    def place_ring(self, kind: str, members: tuple[int, ...], sid: int, length: int) -> None:
        g = len(members)
        ranges = ranges_from_sizes(balanced_zigzag_sizes(length, g, [self.running[r] for r in members]))
        occupied = [i for i, rs in enumerate(ranges) if rs]
        ranks = {members[i] for i in occupied}
        if len(ranks) < 2:
            # too short to occupy two ranks: run it locally
            self.place_whole(sid, length, members[occupied[0]] if occupied else members[0])
            return
        nodes = {r // self.p for r in ranks}
        if kind == INTER_NODE and len(nodes) == 1:
            # too short to cross nodes: lay it out on that node's members only
            node = next(iter(nodes))
            self.place_ring(INTRA_NODE, tuple(r for r in members if r // self.p == node), sid, length)
            return
        self.zone_of[sid] = kind
        self.rings.setdefault((kind, members), []).append(
            RingSequence(sequence_id=sid, ranges_by_position=tuple(tuple(r) for r in ranges)))
        for pos, rank in enumerate(members):
            for a, b in ranges[pos]:
                self.fragments[rank].append(Fragment(sid, a, b, rank))
                self.running[rank] += b - a


def _assemble(batch, cluster: ClusterSpec, inter: InterNodeAssignment,
              intra: list[IntraNodeAssignment], attempt: int) -> PlacementPlan:
    lengths = batch.lengths
    p = cluster.gpus_per_node
    lay = _Layout(cluster)
    jobs: list[tuple[str, tuple[int, ...], int, int]] = []

    nodes_of: dict[int, list[int]] = {}
    for n, bucket in enumerate(inter.buckets):
        for c in bucket.chunks:
            nodes_of.setdefault(c.sequence_id, []).append(n)
    for sid in sorted(nodes_of):
        spanned = sorted(set(nodes_of[sid]))
        if len(spanned) >= 2:
            jobs.append((INTER_NODE, tuple(r for n in spanned for r in cluster.ranks_of_node(n)), sid, lengths[sid]))
        elif p >= 2:
            jobs.append((INTRA_NODE, tuple(cluster.ranks_of_node(spanned[0])), sid, lengths[sid]))
        else:
            lay.place_whole(sid, lengths[sid], spanned[0] * p)

    for n, assignment in enumerate(intra):
        devs_of: dict[int, list[int]] = {}
        for dev, entries in enumerate(assignment.devices):
            for e in entries:
                if e.kind != "chunk_part":  # chunks were handled at node level
                    devs_of.setdefault(e.sequence_id, []).append(dev)
        for sid in sorted(devs_of):
            devs = sorted(set(devs_of[sid]))
            if len(devs) >= 2:
                jobs.append((INTRA_NODE, tuple(n * p + d for d in devs), sid, lengths[sid]))
            else:
                lay.place_whole(sid, lengths[sid], n * p + devs[0])

    # narrow rings first: they have the least placement freedom
    lay.running = [sum(f.tokens for f in frs) for frs in lay.fragments]
    for kind, members, sid, length in sorted(jobs, key=lambda j: (len(j[1]), j[1], j[2])):
        lay.place_ring(kind, members, sid, length)

    rings = tuple(RingGroup(kind=kind, members=members,
                            sequences=tuple(sorted(seqs, key=lambda s: s.sequence_id)))
                  for (kind, members), seqs in sorted(lay.rings.items()))
    for frs in lay.fragments:
        frs.sort(key=lambda f: (f.micro_batch, f.sequence_id, f.start))
    node_buckets = []
    for n in range(cluster.num_nodes):
        acc: dict[int, int] = {}
        for r in cluster.ranks_of_node(n):
            for f in lay.fragments[r]:
                acc[f.sequence_id] = acc.get(f.sequence_id, 0) + f.tokens
        node_buckets.append(sorted(acc.items()))
    return PlacementPlan(
        strategy="zeppelin",
        num_nodes=cluster.num_nodes,
        gpus_per_node=p,
        s1=inter.s1,
        s0_per_node=[a.s0 for a in intra],
        zone_of=lay.zone_of,
        sequence_lengths=dict(lengths),
        node_buckets=node_buckets,
        fragments=lay.fragments,
        ring_groups=rings,
        tokens_per_rank=[sum(f.tokens for f in frs) for frs in lay.fragments],
        micro_batch_counts=[1] * cluster.num_ranks,
        meta={"s1_restarts": inter.restarts, "s0_restarts": [a.restarts for a in intra],
              "reconcile_attempts": attempt},
    )


# ----------------------------------------------------------------- checks & I/O

def validate_plan(plan: PlacementPlan, batch, cluster: ClusterSpec) -> None:
    lengths = batch.lengths
    if set(plan.sequence_lengths) != set(lengths):
        raise PlanValidationError("plan covers a different sequence id set than the batch")
    if plan.total_tokens() != batch.total_tokens:
        raise PlanValidationError("token conservation violated")
    spans: dict[int, list[tuple[int, int]]] = {sid: [] for sid in lengths}
    ranks_of: dict[int, set[int]] = {sid: set() for sid in lengths}
    for rank, frs in enumerate(plan.fragments):
        for f in frs:
            if f.rank != rank:
                raise PlanValidationError("fragment filed under the wrong rank")
            spans[f.sequence_id].append((f.start, f.end))
            ranks_of[f.sequence_id].add(rank)
    for sid, rs in spans.items():
        at = 0
        for a, b in sorted(rs):
            if a != at or b <= a:
                raise PlanValidationError(f"sequence {sid} fragments do not tile [0, {lengths[sid]})")
            at = b
        if at != lengths[sid]:
            raise PlanValidationError(f"sequence {sid} fragments do not cover its length")
    bad = first_over_capacity(plan, cluster)
    if bad is not None:
        raise PlanValidationError(f"rank {bad} exceeds token capacity")
    for sid, zone in plan.zone_of.items():
        ranks = ranks_of.get(sid) or {f.rank for frs in plan.fragments for f in frs if f.sequence_id == sid}
        nodes = {cluster.node_of(r) for r in ranks}
        if zone == LOCAL and len(ranks) != 1:
            raise PlanValidationError(f"local sequence {sid} spans {len(ranks)} ranks")
        if zone == INTRA_NODE and (len(nodes) != 1 or len(ranks) < 2):
            raise PlanValidationError(f"intra-node sequence {sid} has a bad span")
        if zone == INTER_NODE and len(nodes) < 2:
            raise PlanValidationError(f"inter-node sequence {sid} stays within one node")
    for ring in plan.ring_groups:
        nodes = {cluster.node_of(r) for r in ring.members}
        if ring.kind == INTER_NODE and len(nodes) < 2:
            raise PlanValidationError("inter-node ring does not span nodes")
        if ring.kind == INTRA_NODE and len(nodes) != 1:
            raise PlanValidationError("intra-node ring crosses nodes")


def plan_to_json(plan: PlacementPlan) -> str:
    """Canonical plan text (indent=1, sorted keys): the bit-exact comparator."""
    doc = {
        "strategy": plan.strategy,
        "num_nodes": plan.num_nodes,
        "gpus_per_node": plan.gpus_per_node,
        "s1": plan.s1,
        "s0_per_node": plan.s0_per_node,
        "zones": {str(k): plan.zone_of[k] for k in sorted(plan.zone_of)},
        "sequence_lengths": {str(k): plan.sequence_lengths[k] for k in sorted(plan.sequence_lengths)},
        "node_buckets": [[[sid, tok] for sid, tok in nb] for nb in plan.node_buckets],
        "ranks": [[{"sequence_id": f.sequence_id, "start": f.start, "end": f.end,
                    "micro_batch": f.micro_batch} for f in frs] for frs in plan.fragments],
        "rings": [{"kind": r.kind, "members": list(r.members),
                   "sequences": [{"sequence_id": s.sequence_id,
                                  "ranges": [[list(x) for x in pos] for pos in s.ranges_by_position]}
                                 for s in r.sequences]}
                  for r in plan.ring_groups],
        "micro_batch_counts": plan.micro_batch_counts,
        "meta": plan.meta,
    }
    return json.dumps(doc, indent=1, sort_keys=True)


def plan_from_json(text: str) -> PlacementPlan:
    doc = json.loads(text)
    try:
        fragments = [[Fragment(e["sequence_id"], e["start"], e["end"], rank, e.get("micro_batch", 0))
                      for e in frs] for rank, frs in enumerate(doc["ranks"])]
        rings = tuple(
            RingGroup(kind=r["kind"], members=tuple(r["members"]),
                      sequences=tuple(RingSequence(sequence_id=s["sequence_id"],
                                                   ranges_by_position=tuple(tuple(tuple(x) for x in pos)
                                                                            for pos in s["ranges"]))
                                      for s in r["sequences"]))
            for r in doc["rings"])
        return PlacementPlan(
            strategy=doc["strategy"],
            num_nodes=doc["num_nodes"],
            gpus_per_node=doc["gpus_per_node"],
            s1=doc["s1"],
            s0_per_node=list(doc["s0_per_node"]),
            zone_of={int(k): v for k, v in doc["zones"].items()},
            sequence_lengths={int(k): v for k, v in doc["sequence_lengths"].items()},
            node_buckets=[[(sid, tok) for sid, tok in nb] for nb in doc["node_buckets"]],
            fragments=fragments,
            ring_groups=rings,
            tokens_per_rank=[sum(f.tokens for f in frs) for frs in fragments],
            micro_batch_counts=list(doc["micro_batch_counts"]),
            meta=dict(doc.get("meta", {})),
        )
    except (KeyError, TypeError) as exc:
        raise ValueError(f"malformed plan file: missing or invalid key ({exc})") from exc


def save_plan(path: str, plan: PlacementPlan) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(plan_to_json(plan) + "\n")


def load_plan(path: str) -> PlacementPlan:
    with open(path, "r", encoding="utf-8") as fh:
        return plan_from_json(fh.read())


def batch_from_plan(plan: PlacementPlan):
    from .batch import SequenceBatch
    return SequenceBatch(tuple(sorted(plan.sequence_lengths.items())))
