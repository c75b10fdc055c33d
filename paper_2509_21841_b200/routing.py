"""Ring-transfer routing.

Across nodes the reference decomposes a ring send into dispatch / multi-NIC
transfer / combine over proxy ranks (``routing.py:59-185``).  Inside one
NVSwitch box every GPU reaches every peer at full bandwidth, so for the
single-node plans this framework executes ``route_schedule`` returns ``{}``
(reference ``routing.py:171-173``) and "routing" reduces to ordering ring
transfers so that each GPU is one-in / one-out per round — which the ring
executor in ``engine.py`` guarantees by construction.  The cross-node API is
kept (same names, same numbers) so multi-node plans still drop in.
"""

from __future__ import annotations

from dataclasses import dataclass

from .cluster import ClusterSpec
from .schedule import INTER_NODE, AttentionSchedule, RingGroup, split_even

DISPATCH = "dispatch"
INTER_TRANSFER = "inter_transfer"
COMBINE = "combine"


@dataclass(frozen=True)
class RouteStep:
    kind: str
    source_rank: int
    dest_rank: int
    tokens: int
    scope: str


@dataclass(frozen=True)
class RoutePlan:
    source_rank: int
    dest_rank: int
    tokens: int
    x1: int
    x2: int
    send_proxies: tuple[int, ...]
    recv_proxies: tuple[int, ...]
    steps: tuple[RouteStep, ...]
    dispatch_time: float
    transfer_time: float
    combine_time: float

    @property
    def routed_time(self) -> float:
        return self.dispatch_time + self.transfer_time + self.combine_time


def routed_time(cluster: ClusterSpec, n, x1: int, x2: int) -> float:
    """Eq. 2: b_intra*n*(x1-1)/x1 + b_inter*max(n/x1, n/x2) + b_intra*n*(x2-1)/x2."""
    if n < 0:
        raise ValueError("token count must be >= 0")
    if x1 < 1 or x2 < 1:
        raise ValueError("proxy counts must be >= 1")
    bi, be = cluster.inv_bw_intra, cluster.inv_bw_inter
    return bi * n * (x1 - 1) / x1 + be * max(n / x1, n / x2) + bi * n * (x2 - 1) / x2


def _proxy_order(cluster: ClusterSpec, ring: RingGroup, node: int, endpoint: int) -> list[int]:
    ranks = list(cluster.ranks_of_node(node))
    ordered = [r for r in ranks if r in ring.members] + [r for r in ranks if r not in ring.members]
    ordered.remove(endpoint)
    return [endpoint] + ordered


def select_proxies(cluster: ClusterSpec, ring: RingGroup, source_rank: int, dest_rank: int,
                   available: dict[int, int] | None = None):
    a, b = cluster.node_of(source_rank), cluster.node_of(dest_rank)
    if a == b:
        raise ValueError("proxy selection applies to cross-node transfers only")
    p = cluster.gpus_per_node
    avail = available or {}
    na, nb = min(avail.get(a, p), p), min(avail.get(b, p), p)
    x1 = max(1, min(na, nb))
    x2 = max(1, min(nb, na))
    return (x1, x2, tuple(_proxy_order(cluster, ring, a, source_rank)[:x1]),
            tuple(_proxy_order(cluster, ring, b, dest_rank)[:x2]))


def build_route(cluster: ClusterSpec, ring: RingGroup, source_rank: int, dest_rank: int,
                tokens: int, available: dict[int, int] | None = None) -> RoutePlan:
    x1, x2, sp, rp = select_proxies(cluster, ring, source_rank, dest_rank, available)
    steps = [RouteStep(DISPATCH, source_rank, px, share, "intra")
             for px, share in zip(sp[1:], split_even(tokens, x1)[1:])]
    steps += [RouteStep(INTER_TRANSFER, sp[i % x1], rp[i % x2], share, "inter")
              for i, share in enumerate(split_even(tokens, max(x1, x2)))]
    steps += [RouteStep(COMBINE, px, dest_rank, share, "intra")
              for px, share in zip(rp[1:], split_even(tokens, x2)[1:])]
    bi, be = cluster.inv_bw_intra, cluster.inv_bw_inter
    return RoutePlan(source_rank=source_rank, dest_rank=dest_rank, tokens=tokens, x1=x1, x2=x2,
                     send_proxies=sp, recv_proxies=rp, steps=tuple(steps),
                     dispatch_time=bi * tokens * (x1 - 1) / x1,
                     transfer_time=be * max(tokens / x1, tokens / x2),
                     combine_time=bi * tokens * (x2 - 1) / x2)


def route_schedule(schedule: AttentionSchedule, plan, cluster: ClusterSpec) -> dict:
    """RoutePlan per cross-node send, keyed (ring index, round, source rank);
    empty for single-node plans."""
    routes: dict[tuple[int, int, int], RoutePlan] = {}
    for idx, rs in enumerate(schedule.rings()):
        ring = rs.ring
        if ring.kind != INTER_NODE:
            continue
        g = ring.group_size
        for r in range(g):
            for pos in range(g):
                src, dst = ring.members[pos], ring.members[(pos + 1) % g]
                n = rs.rounds[pos][r].comm_tokens
                if cluster.node_of(src) != cluster.node_of(dst) and n:
                    routes[(idx, r, src)] = build_route(cluster, ring, src, dst, n)
    return routes
