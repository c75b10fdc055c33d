"""Per-rank execution program: plan + schedule -> device work lists.

Pure host logic (integers only), shared by the CUDA executor (``engine.py``)
and the multi-process CPU tests.  For one rank it fixes

* the attention layout: the rank's fragments in plan order (reference
  ``partitioner.py:579-580``), each a contiguous run of rows;
* the LocalTask work list (``attention_engine.py:260-265``);
* for every ring the rank belongs to, in ``schedule.rings()`` order
  (``attention_engine.py:266-271``): the ring KV buffer layout of every
  position, the rows this rank packs into its own buffer, the send / receive
  peers (KV moves position i -> i+1, ``attention_engine.py:247-251``) and one
  work list per round against the KV held from position (i - r) mod g
  (``attention_engine.py:229-244``), with partial-state flags so the rounds
  compose into one exact online softmax;
* the remap permutation (``remap.RemapLayout``).

Every per-round work list's exact pair count is checked against the
schedule's ``compute_pairs`` when the program is built.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .remap import RemapLayout, remap_layout
from .schedule import LOCAL, AttentionSchedule, RingSchedule, ring_source
from .worklist import (ITEM_LOAD_STATE, ITEM_STORE_STATE, BwdWorkList, QueryFragment, WorkList,
                       build_bwd_worklist, build_worklist, tile_visible_pairs, TILE)


@dataclass
class RingRoundProgram:
    round_index: int
    src_position: int
    kv_rows: int            # rows of the KV set held this round
    work: WorkList
    frags: list[QueryFragment] = field(default_factory=list)  # query fragments vs the held KV
    # round 0 only (the position's own KV set): the same items with segments in
    # attention-layout rows, so the round reads k / v in place while the set
    # is packed for the successor
    work_in_place: WorkList | None = None


@dataclass
class RingProgram:
    ring_index: int                     # index in schedule.rings()
    members: tuple[int, ...]
    position: int
    next_rank: int
    prev_rank: int
    held_rows: list[int]                # KV rows held by each position
    pack_ranges: np.ndarray             # int32 [n, 3]: (buf_row, layout_row, n_rows)
    state_rows: int                     # partial-state rows this rank needs for the ring
    rounds: list[RingRoundProgram] = field(default_factory=list)

    @property
    def group_size(self) -> int:
        return len(self.members)

    def send_rows(self, round_index: int) -> int:
        """Rows forwarded to next_rank after round ``round_index``."""
        return self.held_rows[ring_source(self.position, round_index, self.group_size)]

    def recv_rows(self, round_index: int) -> int:
        """Rows arriving from prev_rank for round ``round_index + 1``."""
        return self.held_rows[ring_source(self.position, round_index + 1, self.group_size)]

    @property
    def n_buffers(self) -> int:
        """KV buffers per rank: three for rings of 3+ members (a set waits only
        for the round two rounds back to free its buffer), two otherwise."""
        return 3 if self.group_size > 2 else 2

    def hops(self) -> list["RingHop"]:
        """The pull protocol of this position's g-1 hops (see RingHop)."""
        g, nb = self.group_size, self.n_buffers
        return [RingHop(round_index=r, src_buf=r % nb, dst_buf=(r + 1) % nb, rows=self.recv_rows(r),
                        full=r, free=(r + 1 - nb) if r + 1 - nb >= 0 else None, consumed=r,
                        next_full=(r + 1) if r + 1 <= g - 2 else None)
                for r in range(g - 1)]


@dataclass(frozen=True)
class RingHop:
    """Hop r of a ring position (reference attention_engine.py:247-251: after
    round r the KV set held at position i-1 moves to position i), executed as
    a pull by position i.  Epoch fields are offsets r' of the ring's epoch
    base E: flags carry E + r'.

    * wait until the predecessor announced ``full`` (its buffer ``src_buf``
      holds the set for this position's round r+1);
    * if ``free`` is set, wait until the successor announced it consumed hop
      ``free`` from this rank (``dst_buf``'s previous content); the compute
      stream also waits for round r+1-n_buffers, the buffer's last reader;
    * copy ``rows`` KV rows predecessor[src_buf] -> own[dst_buf];
    * announce ``consumed`` to the predecessor and, if ``next_full`` is set,
      announce ``next_full`` to the successor (own ``dst_buf`` is what it
      pulls at its hop r+1).

    Position i's own set is packed into buffer 0 and announced to the
    successor with epoch offset 0 before the first round.  A flag only grows:
    a rank leaves a ring after its successor consumed its last hop, so no
    epoch of a later ring can satisfy a wait of an earlier one."""
    round_index: int
    src_buf: int
    dst_buf: int
    rows: int
    full: int
    free: int | None
    consumed: int
    next_full: int | None


@dataclass
class RankProgram:
    rank: int
    world: int
    rows: int                           # A_rank, attention-layout rows
    frag_rows: dict[tuple[int, int], int]  # (sid, start) -> layout row
    local: WorkList
    rings: list[RingProgram]
    remap: RemapLayout
    n_head_pairs: int
    local_frags: list[QueryFragment] = field(default_factory=list)
    # local items [cuts[j-1], cuts[j]) run right before the j-th ring of this
    # rank (cuts[-1] before the first); the rest after the last ring
    local_cuts: list[int] = field(default_factory=list)

    def pairs_per_head(self) -> int:
        return self.local.pairs_per_head + sum(rr.work.pairs_per_head for r in self.rings for rr in r.rounds)


def _ring_buffer_rows(ring_sched: RingSchedule) -> list[dict[tuple[int, int], int]]:
    """Per position: (sid, start) -> row in that position's KV buffer
    (sequences by id, ranges in order)."""
    ring = ring_sched.ring
    out = []
    for p in range(ring.group_size):
        at, rows = 0, {}
        for seq in ring.sequences:
            for a, b in seq.ranges_by_position[p]:
                rows[(seq.sequence_id, a)] = at
                at += b - a
        out.append(rows)
    return out


def local_fill_plan(schedule: AttentionSchedule, num_ranks: int) -> dict[int, list[int]]:
    """Local work (visible pairs per head) each rank runs before each of its
    rings, so that LocalTasks fill the time a rank would otherwise wait for a
    ring's slowest member.

    The reference's executor model (simulator.py:136-187): rings run in
    schedule order, a ring starts when all its members are ready (:139), local
    tasks run after the rings (:181-187).  Here the same list schedule is
    played with exact pair counts as the cost: at each ring, a member that
    would be idle until the ring's start runs that much of its local work
    first (longest tiles first); whatever local work is left runs after its
    last ring.  Pure function of the schedule, so every rank derives the same
    plan.  Returns rank -> [pairs before its 1st ring, before its 2nd, ...]."""
    in_ring = {s.sequence_id for rs in schedule.rings() for s in rs.ring.sequences}
    local_left = [0] * num_ranks
    for t in schedule.local_tasks:
        if t.sequence_id not in in_ring:
            local_left[t.rank] += t.compute_pairs
    ready = [0] * num_ranks
    fill: dict[int, list[int]] = {r: [] for r in range(num_ranks)}
    for rs in schedule.rings():
        members = rs.ring.members
        start = max(ready[m] for m in members)
        for m in members:
            take = min(start - ready[m], local_left[m])
            fill[m].append(take)
            local_left[m] -= take
        work = [sum(rd.compute_pairs for rd in rs.rounds[i]) for i in range(len(members))]
        end = start + max(work)
        for m in members:
            ready[m] = end
    return fill


def build_rank_program(plan, schedule: AttentionSchedule, rank: int, n_heads: int,
                       remap=None) -> RankProgram:
    n_hp = n_heads // 2
    frag_rows: dict[tuple[int, int], int] = {}
    at = 0
    local_frags: list[QueryFragment] = []
    # A sequence that rides a ring is computed by its ring rounds only.  (The
    # even-split baselines label a short ring member LOCAL when it lands on one
    # rank; the reference cost model then charges it twice, execution must not.)
    in_ring = {s.sequence_id for rs in schedule.rings() for s in rs.ring.sequences}
    for f in plan.fragments[rank]:
        frag_rows[(f.sequence_id, f.start)] = at
        if (plan.zone_of.get(f.sequence_id) == LOCAL or f.micro_batch > 0) and f.sequence_id not in in_ring:
            local_frags.append(QueryFragment(row0=at, pos0=0, length=f.tokens, segs=[(at, 0, f.tokens)]))
        at += f.tokens
    local = build_worklist(local_frags, n_hp)
    # local items run before each ring (cumulative cut points in the LPT list)
    cuts, acc = [], 0
    for take in local_fill_plan(schedule, plan.num_ranks)[rank]:
        acc += take
        cuts.append(local.cut(acc))
    want = sum(t.compute_pairs for t in schedule.local_tasks if t.rank == rank and t.sequence_id not in in_ring)
    if local.pairs_per_head != want:
        raise AssertionError(f"rank {rank}: local work list covers {local.pairs_per_head} pairs, schedule says {want}")

    rings: list[RingProgram] = []
    for ri, rs in enumerate(schedule.rings()):
        ring = rs.ring
        if rank not in ring.members:
            continue
        g = ring.group_size
        i = ring.members.index(rank)
        buf_rows = _ring_buffer_rows(rs)
        held = [ring.kv_tokens(p) for p in range(g)]
        pack = [(buf_rows[i][(s.sequence_id, a)], frag_rows[(s.sequence_id, a)], b - a)
                for s in ring.sequences for a, b in s.ranges_by_position[i]]
        # this rank's query fragments of the ring, with compact state rows
        qf: list[tuple[int, int, int, int, int]] = []  # (sid, layout_row, pos0, len, state_row0)
        srow = 0
        for s in ring.sequences:
            for a, b in s.ranges_by_position[i]:
                qf.append((s.sequence_id, frag_rows[(s.sequence_id, a)], a, b - a, srow))
                srow += b - a
        seq_by_id = {s.sequence_id: s for s in ring.sequences}

        def segs_for(sid: int, src: int) -> list[tuple[int, int, int]]:
            return [(buf_rows[src][(sid, c)], c, d - c) for c, d in seq_by_id[sid].ranges_by_position[src]]

        # visibility of every query tile in every round -> first / last round
        vis = []
        for sid, _, a, n, _ in qf:
            p0 = a + np.arange(0, n, TILE)
            ln = np.minimum(TILE, n - np.arange(0, n, TILE))
            vis.append(np.stack([tile_visible_pairs(p0, ln, segs_for(sid, ring_source(i, r, g))) > 0
                                 for r in range(g)]))
        prog = RingProgram(ring_index=ri, members=ring.members, position=i,
                           next_rank=ring.members[(i + 1) % g], prev_rank=ring.members[(i - 1) % g],
                           held_rows=held, pack_ranges=np.asarray(pack, dtype=np.int32).reshape(-1, 3),
                           state_rows=srow)
        for r in range(g):
            src = ring_source(i, r, g)
            frags = [QueryFragment(row0=row, pos0=a, length=n, segs=segs_for(sid, src), state_row0=st)
                     for sid, row, a, n, st in qf]

            def flags(fi, p0, ln, r=r):
                v = vis[fi]
                seen_before = v[:r].any(axis=0)
                seen_after = v[r + 1:].any(axis=0)
                return np.where(seen_before, ITEM_LOAD_STATE, 0) | np.where(seen_after, ITEM_STORE_STATE, 0)

            wl = build_worklist(frags, n_hp, tile_flags=flags)
            expect = rs.rounds[i][r].compute_pairs
            if wl.pairs_per_head != expect:
                raise AssertionError(f"rank {rank} ring {ring.members} round {r}: work list covers "
                                     f"{wl.pairs_per_head} pairs, schedule says {expect}")
            in_place = None
            if src == i:
                own = [QueryFragment(row0=f.row0, pos0=f.pos0, length=f.length, state_row0=f.state_row0,
                                     segs=[(frag_rows[(sid, c)], c, d - c)
                                           for c, d in seq_by_id[sid].ranges_by_position[i]])
                       for (sid, _, _, _, _), f in zip(qf, frags)]
                in_place = build_worklist(own, n_hp, tile_flags=flags)
                if in_place.pairs_per_head != expect:
                    raise AssertionError(f"rank {rank} ring {ring.members}: in-place round 0 covers "
                                         f"{in_place.pairs_per_head} pairs, schedule says {expect}")
            prog.rounds.append(RingRoundProgram(round_index=r, src_position=src, kv_rows=held[src], work=wl,
                                                work_in_place=in_place,
                                                frags=frags))
        rings.append(prog)

    if remap is None:
        remap = remap_layout(plan.tokens_per_rank)
    elif not isinstance(remap, RemapLayout):
        remap = remap_layout(plan.tokens_per_rank, remap)
    return RankProgram(rank=rank, world=plan.num_ranks, rows=at, frag_rows=frag_rows, local=local,
                       rings=rings, remap=remap, n_head_pairs=n_hp, local_frags=local_frags, local_cuts=cuts)


@dataclass
class BwdProgram:
    """Backward work lists of a RankProgram (``zp_attn_bwd``): the LocalTask
    list and one list per ring round, each covering exactly the forward's
    visible pairs (checked), plus the row tables that return a ring's dK/dV
    from its KV buffer to the attention layout."""
    local: BwdWorkList
    rounds: list[list[BwdWorkList]]      # [ring][round]
    unpack_ranges: list[np.ndarray]      # [ring]: int32 [n, 3] (layout_row, buf_row, n_rows)


def build_bwd_program(prog: RankProgram, n_kv_heads: int) -> BwdProgram:
    local = build_bwd_worklist(prog.local_frags, n_kv_heads)
    if local.pairs_per_head != prog.local.pairs_per_head:
        raise AssertionError(f"rank {prog.rank}: backward local list covers {local.pairs_per_head} pairs, "
                             f"forward {prog.local.pairs_per_head}")
    rounds = []
    for rp in prog.rings:
        lists = []
        for rr in rp.rounds:
            wl = build_bwd_worklist(rr.frags, n_kv_heads)
            if wl.pairs_per_head != rr.work.pairs_per_head:
                raise AssertionError(f"rank {prog.rank} ring {rp.members} round {rr.round_index}: backward list "
                                     f"covers {wl.pairs_per_head} pairs, forward {rr.work.pairs_per_head}")
            lists.append(wl)
        rounds.append(lists)
    unpack = [np.ascontiguousarray(rp.pack_ranges[:, [1, 0, 2]]) for rp in prog.rings]
    return BwdProgram(local=local, rounds=rounds, unpack_ranges=unpack)
