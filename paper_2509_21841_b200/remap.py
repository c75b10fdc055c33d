"""Attention <-> linear token remapping: transfer matrix + row permutation.

Two halves:

1. ``solve_remap`` — the minimax transfer matrix M (rows: surplus senders,
   columns: deficit receivers) of the reference (``remapping.py:29-245``):
   bisection on the per-sender cost bound, each bound checked by an
   Edmonds-Karp max flow whose arcs are inserted in the reference's order, so
   the integer matrix (and the float objective) are identical.  On one NVSwitch
   box every off-diagonal cost is equal and M reduces to the northwest-corner
   rule over (senders ascending x receivers ascending) — ``northwest_corner``
   is kept as an independent check, not as a replacement.

2. ``RemapLayout`` — the row-level permutation that moves data (R3 in
   SURVEY.md; the reference pins only the counts).  Rank i's attention layout
   is its fragments in plan order; it keeps rows [0, min(A_i, B_i)) and sends
   its tail [B_i, A_i) to receivers j ascending, M[i][j] rows each.  Receiver
   j's linear layout is its kept rows followed by received blocks in
   sender-ascending order.  The inverse is the exact reverse.  Because both
   the send tail and the receive region are contiguous, the device path moves
   them without any gather (NCCL all-to-allv on slices, or direct peer
   stores), see ``engine.py``.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

from .cluster import ClusterSpec

_EPS = 1e-9


def target_distribution(counts: list[int]) -> list[int]:
    d = len(counts)
    if d < 1:
        raise ValueError("need at least one rank")
    if any(c < 0 for c in counts):
        raise ValueError("token counts must be >= 0")
    q, r = divmod(sum(counts), d)
    # all fractional parts are equal, so the remainder goes to the lowest indices
    return [q + (i < r) for i in range(d)]


def cost_matrix(cluster: ClusterSpec) -> np.ndarray:
    d = cluster.num_ranks
    node = np.arange(d) // cluster.gpus_per_node
    t = np.where(node[:, None] == node[None, :], cluster.inv_bw_intra, cluster.inv_bw_inter).astype(float)
    np.fill_diagonal(t, 0.0)
    return t


@dataclass(frozen=True)
class RemapResult:
    matrix: np.ndarray     # int64 d x d token transfers
    objective: float       # continuous minimax optimum
    row_costs: np.ndarray  # per-sender cost of the integer matrix
    col_costs: np.ndarray  # per-receiver cost (diagnostic)


class _FlowNet:
    """Residual graph with paired arcs (arc e, reverse e^1) and BFS augmenting
    paths (Edmonds-Karp); capacities are floats."""

    def __init__(self, n: int):
        self.adj: list[list[int]] = [[] for _ in range(n)]
        self.head: list[int] = []
        self.res: list[float] = []

    def arc(self, u: int, v: int, cap: float) -> int:
        e = len(self.head)
        self.adj[u].append(e)
        self.head.append(v)
        self.res.append(cap)
        self.adj[v].append(e + 1)
        self.head.append(u)
        self.res.append(0.0)
        return e

    def flow_on(self, e: int) -> float:
        return self.res[e ^ 1]

    def maxflow(self, s: int, t: int) -> float:
        total = 0.0
        n = len(self.adj)
        while True:
            via = [-1] * n
            via[s] = -2
            frontier = deque([s])
            while frontier and via[t] == -1:
                u = frontier.popleft()
                for e in self.adj[u]:
                    w = self.head[e]
                    if via[w] == -1 and self.res[e] > _EPS:
                        via[w] = e
                        frontier.append(w)
            if via[t] == -1:
                return total
            path = []
            w = t
            while w != s:
                e = via[w]
                path.append(e)
                w = self.head[e ^ 1]
            push = float("inf")
            for e in path:
                push = min(push, self.res[e])
            for e in path:
                self.res[e] -= push
                self.res[e ^ 1] += push
            total += push


def _two_costs(row: np.ndarray, receivers: list[int]) -> tuple[float, float]:
    levels = sorted({float(row[j]) for j in receivers})
    if len(levels) > 2:
        raise ValueError("cost matrix rows may carry at most two distinct arc costs")
    return levels[0], levels[-1]


def _bound_feasible(senders, receivers, u, v, t, bound: float, integral: bool):
    """Flow {(i, j): amount} meeting every sender's cost bound, or None.

    Network: source -> sender i (cap u_i); sender -> its budget node (cap =
    tokens it may push over expensive arcs under ``bound``); cheap arcs leave
    the sender, expensive arcs leave the budget node; receiver j -> sink
    (cap v_j)."""
    ns = len(senders)
    net = _FlowNet(2 + 2 * ns + len(receivers))
    src, sink = 0, 1
    snode = {i: 2 + k for k, i in enumerate(senders)}
    bnode = {i: 2 + ns + k for k, i in enumerate(senders)}
    rnode = {j: 2 + 2 * ns + k for k, j in enumerate(receivers)}
    big = float(u.sum())
    arcs: dict[tuple[int, int], int] = {}
    for i in senders:
        net.arc(src, snode[i], float(u[i]))
        cheap, dear = _two_costs(t[i], receivers)
        if cheap * u[i] > bound * (1 + _EPS) + _EPS:
            return None
        budget = (bound - cheap * float(u[i])) / (dear - cheap) if dear > cheap else big
        if integral:
            budget = float(np.floor(budget + _EPS))
        net.arc(snode[i], bnode[i], max(0.0, budget))
        for j in receivers:
            start = snode[i] if float(t[i][j]) <= cheap + _EPS else bnode[i]
            arcs[(i, j)] = net.arc(start, rnode[j], big)
    for j in receivers:
        net.arc(rnode[j], sink, float(v[j]))
    need = float(u.sum())
    if net.maxflow(src, sink) + max(1e-9, 1e-12 * need) < need:
        return None
    return {key: net.flow_on(e) for key, e in arcs.items()}


def _bisect(lo: float, hi: float, ok) -> float:
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if ok(mid):
            hi = mid
        else:
            lo = mid
        if hi - lo <= 1e-9 * max(hi, 1e-30):
            break
    return hi


def solve_remap(counts: list[int], cost: np.ndarray) -> RemapResult:
    a = np.asarray(counts, dtype=np.int64)
    d = len(a)
    t = np.asarray(cost, dtype=float)
    if t.shape != (d, d):
        raise ValueError("cost matrix shape does not match the rank count")
    b = np.asarray(target_distribution(list(counts)), dtype=np.int64)
    u = np.maximum(a - b, 0)
    v = np.maximum(b - a, 0)
    matrix = np.zeros((d, d), dtype=np.int64)
    if u.sum() == 0:
        zero = np.zeros(d)
        return RemapResult(matrix=matrix, objective=0.0, row_costs=zero, col_costs=zero)
    senders = [i for i in range(d) if u[i] > 0]
    receivers = [j for j in range(d) if v[j] > 0]

    def feasible(bound: float, integral: bool):
        return _bound_feasible(senders, receivers, u, v, t, bound, integral)

    hi = max(float(u[i]) * float(max(t[i][j] for j in receivers)) for i in senders)
    objective = _bisect(0.0, hi, lambda x: feasible(x, False) is not None)
    # integral matrix: floor the budgets, smallest bound still saturating
    if feasible(objective, True) is None:
        bound = _bisect(objective, objective + 2.0 * float(t.max()) + 1.0,
                        lambda x: feasible(x, True) is not None)
    else:
        bound = objective
    flow = feasible(bound, True)
    assert flow is not None
    for (i, j), amount in flow.items():
        matrix[i][j] = int(round(amount))
    return RemapResult(matrix=matrix, objective=objective,
                       row_costs=(t * matrix).sum(axis=1), col_costs=(t * matrix).sum(axis=0))


def remap_cost_pair(tokens_per_rank: list[int], cluster: ClusterSpec) -> tuple[float, float]:
    """Forward and inverse remap cost; the inverse replays the transfers
    reversed over a symmetric cost matrix (reference remapping.py:248-255)."""
    res = solve_remap(tokens_per_rank, cost_matrix(cluster))
    return res.objective, res.objective


def matrix_to_csv(matrix: np.ndarray) -> str:
    return "".join(",".join(str(int(x)) for x in row) + "\n" for row in matrix)


def northwest_corner(counts: list[int]) -> np.ndarray:
    """Northwest-corner transport plan over (senders asc x receivers asc).
    Equals solve_remap's matrix whenever all off-diagonal costs are equal
    (one node); used as an independent cross-check in tests."""
    a = np.asarray(counts, dtype=np.int64)
    b = np.asarray(target_distribution(list(counts)), dtype=np.int64)
    sup = [[i, int(x)] for i, x in enumerate(np.maximum(a - b, 0)) if x > 0]
    dem = [[j, int(x)] for j, x in enumerate(np.maximum(b - a, 0)) if x > 0]
    m = np.zeros((len(a), len(a)), dtype=np.int64)
    si = di = 0
    while si < len(sup) and di < len(dem):
        q = min(sup[si][1], dem[di][1])
        m[sup[si][0], dem[di][0]] += q
        sup[si][1] -= q
        dem[di][1] -= q
        si += sup[si][1] == 0
        di += dem[di][1] == 0
    return m


@dataclass(frozen=True)
class RemapLayout:
    """Row permutation implied by (A, M): everything a rank needs to move
    rows between its attention layout (A_i rows) and linear layout (B_i)."""

    attn_rows: tuple[int, ...]     # A
    linear_rows: tuple[int, ...]   # B
    matrix: np.ndarray             # M, int64

    @property
    def world(self) -> int:
        return len(self.attn_rows)

    def kept(self, rank: int) -> int:
        return min(self.attn_rows[rank], self.linear_rows[rank])

    def send_counts(self, rank: int) -> list[int]:
        return [int(x) for x in self.matrix[rank]]

    def recv_counts(self, rank: int) -> list[int]:
        return [int(x) for x in self.matrix[:, rank]]

    def send_offsets(self, rank: int) -> list[int]:
        """Attention-layout row where the block for each receiver starts."""
        out, at = [], self.linear_rows[rank]
        for n in self.send_counts(rank):
            out.append(at)
            at += n
        return out

    def recv_offsets(self, rank: int) -> list[int]:
        """Linear-layout row where the block from each sender lands."""
        out, at = [], self.attn_rows[rank]
        for n in self.recv_counts(rank):
            out.append(at)
            at += n
        return out

    def moved_rows(self) -> int:
        return int(self.matrix.sum())

    def forward_slices(self, rank: int):
        """(kept rows, attention-layout rows sent [lo, hi), linear-layout rows
        received [lo, hi), send counts per receiver, recv counts per sender)."""
        a, b = self.attn_rows[rank], self.linear_rows[rank]
        return (min(a, b), (b, max(a, b)), (a, max(a, b)), self.send_counts(rank), self.recv_counts(rank))

    def inverse_slices(self, rank: int):
        """Mirror of forward_slices for the linear -> attention direction:
        (kept, linear rows sent, attention rows received, send counts, recv counts)."""
        a, b = self.attn_rows[rank], self.linear_rows[rank]
        return (min(a, b), (a, max(a, b)), (b, max(a, b)), self.recv_counts(rank), self.send_counts(rank))

    def source_of_linear_rows(self, rank: int) -> list[tuple[int, int, int]]:
        """(src_rank, src_row0, n) blocks composing rank's linear layout, in order."""
        blocks = [(rank, 0, self.kept(rank))] if self.kept(rank) else []
        for s, n in enumerate(self.recv_counts(rank)):
            if n:
                blocks.append((s, self.send_offsets(s)[rank], n))
        return blocks


def remap_layout(counts: list[int], result: RemapResult | None = None,
                 cost: np.ndarray | None = None) -> RemapLayout:
    """Build the row permutation for attention-layout counts A (solving M
    with a uniform cost when no result is given)."""
    counts = [int(c) for c in counts]
    if result is None:
        d = len(counts)
        if cost is None:
            cost = np.ones((d, d)) - np.eye(d)
        result = solve_remap(counts, cost)
    return RemapLayout(attn_rows=tuple(counts), linear_rows=tuple(target_distribution(counts)),
                       matrix=np.asarray(result.matrix, dtype=np.int64))


def identity_layout(counts: list[int]) -> RemapLayout:
    """No remap: the linear modules run on the attention layout (what the
    comparison strategies do; only Zeppelin rebalances)."""
    counts = [int(c) for c in counts]
    return RemapLayout(attn_rows=tuple(counts), linear_rows=tuple(counts),
                       matrix=np.zeros((len(counts), len(counts)), dtype=np.int64))
