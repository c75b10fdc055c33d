"""Host-side work lists for the attention kernel (``zp_attn_fwd``).

A work item is one 128-row query tile of one sequence fragment for one pair
of query heads sharing a KV head.  Items carry the KV segments they attend to
(global in-sequence positions), so the same kernel executes

* LocalTask work: a whole sequence against itself
  (reference ``attention_engine.py:260-265``), and
* one RingRound: a position's query ranges against the KV ranges held by ring
  position ``(i - r) mod g`` (reference ``attention_engine.py:229-244``),

with the causal rule of ``visible_pairs`` (``attention_engine.py:113-136``):
key position <= query position.  Items are sorted longest-first (LPT) so the
hardware block scheduler drains the long causal tiles early.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TILE = 128
# item order: 1 = KV-head-major (default; DRAM 6.0 -> 1.3 GB and +2.5% on config 2), 0 = the head pairs of a tile adjacent (A/B knob)
KV_MAJOR = int(__import__("os").environ.get("ZP_KV_MAJOR", "1"))
BWD_KV_MAJOR = int(__import__("os").environ.get("ZP_BWD_KV_MAJOR", "1"))  # backward list order (1 = KV-head-major; A/B knob)
ITEM_LOAD_STATE = 1
ITEM_STORE_STATE = 2

ITEM_DTYPE = np.dtype([("q_row0", "<i4"), ("q_pos0", "<i4"), ("q_len", "<i4"),
                       ("head_pair", "<i4"), ("seg_begin", "<i4"), ("seg_count", "<i4"),
                       ("state_row0", "<i4"), ("flags", "<i4")])
SEG_DTYPE = np.dtype([("row0", "<i4"), ("pos0", "<i4"), ("len", "<i4"), ("reserved", "<i4")])


@dataclass
class QueryFragment:
    """Query rows [row0, row0+length) holding global positions [pos0, ...),
    attending to KV segments ``segs`` = [(row0, pos0, len), ...] of the same
    sequence.  ``state_row0`` locates the fragment in ring partial-state
    buffers (-1 when unused)."""

    row0: int
    pos0: int
    length: int
    segs: list[tuple[int, int, int]]
    state_row0: int = -1


def kv_tile_counts(max_qpos: np.ndarray, segs: list[tuple[int, int, int]]) -> np.ndarray:
    """Number of 128-key tiles the kernel walks for query tiles whose last
    position is ``max_qpos`` (matches TileCursor in zp_attn.cu)."""
    n = np.zeros_like(max_qpos, dtype=np.int64)
    for _, p0, ln in segs:
        if ln <= 0:
            continue
        vis = np.minimum(ln, max_qpos - p0 + 1)
        n += np.where(max_qpos >= p0, (vis + TILE - 1) // TILE, 0)
    return n


def tile_visible_pairs(q_pos0: np.ndarray, q_len: np.ndarray, segs: list[tuple[int, int, int]]) -> np.ndarray:
    """Exact visible (q,k) pairs per query tile (closed form of visible_pairs,
    reference attention_engine.py:113-136, vectorised over tiles)."""
    a = q_pos0.astype(np.int64)
    b = a + q_len.astype(np.int64)
    total = np.zeros_like(a)
    for _, c, m in segs:
        if m <= 0:
            continue
        d = c + m
        lo = np.maximum(a, c)
        hi = np.minimum(b - 1, d - 2)
        cnt = np.maximum(hi - lo + 1, 0)
        total += np.where(cnt > 0, ((lo + 1 - c) + (hi + 1 - c)) * cnt // 2, 0)
        flat_lo = np.maximum(a, d - 1)
        total += np.maximum(b - flat_lo, 0) * m
    return total


@dataclass
class WorkList:
    items: np.ndarray      # ITEM_DTYPE, sorted longest-first
    segs: np.ndarray       # SEG_DTYPE
    pairs_per_head: int    # visible causal pairs for one query head
    kv_tiles: int          # sum over items of KV tiles walked
    tile_pairs: np.ndarray | None = None  # visible pairs of each item's query tile (one head)
    n_head_pairs: int = 1

    @property
    def n_items(self) -> int:
        return int(self.items.shape[0])

    def cut(self, pairs_per_head: int) -> int:
        """Item index (even: item pairs stay together) such that items
        [0, index) cover about ``pairs_per_head`` visible pairs per head: the
        prefix a rank runs to fill a predicted wait."""
        if pairs_per_head <= 0 or self.tile_pairs is None or not self.n_items:
            return 0
        covered = np.cumsum(self.tile_pairs) / self.n_head_pairs  # pairs per head, item by item
        k = int(np.searchsorted(covered, pairs_per_head, side="left")) + 1
        return min(k + (k & 1), self.n_items)


def build_worklist(frags: list[QueryFragment], n_head_pairs: int,
                   tile_flags=None) -> WorkList:
    """Expand fragments into 128-row tiles x head pairs.

    ``tile_flags(frag_index, tile_q_pos0, tile_len) -> int array`` may attach
    ZP_ITEM_* flags per tile (ring rounds); tiles with no visible pair are
    dropped (they would be pure no-ops)."""
    seg_rows: list[tuple[int, int, int, int]] = []
    cols = {name: [] for name in ("q_row0", "q_pos0", "q_len", "seg_begin", "seg_count",
                                  "state_row0", "flags", "cost")}
    pairs = 0
    for fi, f in enumerate(frags):
        if f.length <= 0:
            continue
        seg_begin = len(seg_rows)
        seg_rows.extend((r, p, n, 0) for r, p, n in f.segs)
        offs = np.arange(0, f.length, TILE, dtype=np.int64)
        q_len = np.minimum(TILE, f.length - offs)
        q_pos0 = f.pos0 + offs
        cost = kv_tile_counts(q_pos0 + q_len - 1, f.segs)
        vis = tile_visible_pairs(q_pos0, q_len, f.segs)
        keep = vis > 0
        if not keep.any():
            continue
        flags = np.zeros_like(offs) if tile_flags is None else np.asarray(tile_flags(fi, q_pos0, q_len))
        pairs += int(vis[keep].sum())
        k = int(keep.sum())
        cols["q_row0"].append(f.row0 + offs[keep])
        cols["q_pos0"].append(q_pos0[keep])
        cols["q_len"].append(q_len[keep])
        cols["seg_begin"].append(np.full(k, seg_begin))
        cols["seg_count"].append(np.full(k, len(f.segs)))
        cols["state_row0"].append((f.state_row0 + offs[keep]) if f.state_row0 >= 0 else np.full(k, -1))
        cols["flags"].append(flags[keep])
        cols["cost"].append(cost[keep])
        cols.setdefault("pairs", []).append(vis[keep])
    segs = np.zeros(max(len(seg_rows), 1), dtype=SEG_DTYPE)
    for i, row in enumerate(seg_rows):
        segs[i] = row
    if not cols["q_row0"]:
        return WorkList(np.zeros(0, dtype=ITEM_DTYPE), segs, 0, 0)
    tiles = {k: np.concatenate(v) for k, v in cols.items()}
    n_tiles = tiles["q_row0"].shape[0]
    order = np.argsort(-tiles["cost"], kind="stable")  # longest tiles first (LPT)
    if KV_MAJOR and n_head_pairs % 2 == 0:
        # KV-head-major: all tiles of head pairs (2g, 2g+1) — one KV head for
        # GQA groups of 4 — longest first, then the next pair of head pairs;
        # the units in flight together stream the same K/V, which then stays
        # in L2 instead of being re-read from HBM
        t_idx = np.tile(np.repeat(order, 2), n_head_pairs // 2)
        hp = (np.repeat(np.arange(0, n_head_pairs, 2), 2 * n_tiles)
              + np.tile(np.array([0, 1]), n_tiles * (n_head_pairs // 2)))
    else:
        # the head pairs of one tile adjacent
        t_idx = np.repeat(order, n_head_pairs)
        hp = np.tile(np.arange(n_head_pairs), n_tiles)
    items = np.zeros(n_tiles * n_head_pairs, dtype=ITEM_DTYPE)
    for name in ("q_row0", "q_pos0", "q_len", "seg_begin", "seg_count", "state_row0", "flags"):
        items[name] = tiles[name][t_idx]
    items["head_pair"] = hp
    kv_tiles = int(tiles["cost"].sum()) * n_head_pairs
    return WorkList(items, segs, pairs, kv_tiles, tiles["pairs"][t_idx], n_head_pairs)


# ------------------------------------------------------------------ backward

BWD_ITEM_DTYPE = np.dtype([("kv_row0", "<i4"), ("kv_pos0", "<i4"), ("kv_len", "<i4"), ("kv_head", "<i4"),
                           ("qseg_begin", "<i4"), ("qseg_count", "<i4"), ("flags", "<i4"),
                           ("reserved", "<i4")])
BWD_ACCUMULATE = 1
BWD_QBLOCK = 64


def kv_tile_visible_pairs(kv_pos0: np.ndarray, kv_len: np.ndarray, qsegs: list[tuple[int, int, int]]) -> np.ndarray:
    """Exact visible (q,k) pairs of key tiles [kv_pos0, +kv_len) against query
    segments (row0, pos0, len) of the same sequence (key position <= query
    position, reference attention_engine.py:113-136), vectorised over tiles."""
    c = kv_pos0.astype(np.int64)
    d = c + kv_len.astype(np.int64)  # keys [c, d)
    total = np.zeros_like(c)
    for _, a, m in qsegs:
        if m <= 0:
            continue
        b = a + m  # queries [a, b)
        # key p sees b - max(a, p) queries when p < b: keys [c, min(d, a+1)) see m each,
        # keys [max(c, a+1), min(d, b)) see b - p
        lo_full = np.minimum(d, a + 1)
        total += np.maximum(lo_full - c, 0) * m
        lo = np.maximum(c, a + 1)
        hi = np.minimum(d, b)  # exclusive
        n = np.maximum(hi - lo, 0)
        total += np.where(n > 0, ((b - lo) + (b - hi + 1)) * n // 2, 0)
    return total


@dataclass
class BwdWorkList:
    items: np.ndarray      # BWD_ITEM_DTYPE, longest-first
    qsegs: np.ndarray      # SEG_DTYPE
    pairs_per_head: int    # visible causal pairs for one query head
    steps: int             # query-block steps summed over items (per GQA group member)

    @property
    def n_items(self) -> int:
        return int(self.items.shape[0])


def build_bwd_worklist(frags: list[QueryFragment], n_kv_heads: int, flags: int = BWD_ACCUMULATE) -> BwdWorkList:
    """Backward work items (``zp_attn_bwd``): every 128-key tile of every KV
    segment the fragments attend to, once per KV head, with the list of query
    fragments that see it.  Fragments sharing a KV segment (the zigzag ranges
    of one sequence in a ring round) are grouped so items cover disjoint key
    tiles."""
    by_seg: dict[tuple[int, int, int], list[tuple[int, int, int]]] = {}
    for f in frags:
        if f.length <= 0:
            continue
        for seg in f.segs:
            if seg[2] > 0:
                by_seg.setdefault(tuple(seg), []).append((f.row0, f.pos0, f.length))
    qrows: list[tuple[int, int, int, int]] = []
    cols = {k: [] for k in ("kv_row0", "kv_pos0", "kv_len", "qseg_begin", "qseg_count", "cost")}
    pairs = 0
    for (r0, p0, ln), qs in sorted(by_seg.items()):
        offs = np.arange(0, ln, TILE, dtype=np.int64)
        kl = np.minimum(TILE, ln - offs)
        kp = p0 + offs
        vis = kv_tile_visible_pairs(kp, kl, qs)
        keep = vis > 0
        if not keep.any():
            continue
        pairs += int(vis[keep].sum())
        begin = len(qrows)
        qrows.extend((a, b, c, 0) for a, b, c in qs)
        # cost: query blocks the kernel walks for each tile
        cost = np.zeros_like(kp)
        for _, a, m in qs:
            first = np.where(kp > a, (kp - a) // BWD_QBLOCK, 0)
            nb = (m + BWD_QBLOCK - 1) // BWD_QBLOCK
            cost += np.where(a + m - 1 >= kp, nb - first, 0)
        k = int(keep.sum())
        cols["kv_row0"].append(r0 + offs[keep])
        cols["kv_pos0"].append(kp[keep])
        cols["kv_len"].append(kl[keep])
        cols["qseg_begin"].append(np.full(k, begin))
        cols["qseg_count"].append(np.full(k, len(qs)))
        cols["cost"].append(cost[keep])
    qsegs = np.zeros(max(len(qrows), 1), dtype=SEG_DTYPE)
    for i, row in enumerate(qrows):
        qsegs[i] = row
    if not cols["kv_row0"]:
        return BwdWorkList(np.zeros(0, dtype=BWD_ITEM_DTYPE), qsegs, 0, 0)
    tiles = {k: np.concatenate(v) for k, v in cols.items()}
    order = np.argsort(-tiles["cost"], kind="stable")
    n_tiles = order.shape[0]
    items = np.zeros(n_tiles * n_kv_heads, dtype=BWD_ITEM_DTYPE)
    if BWD_KV_MAJOR:
        # KV-head-major (longest tiles first within a head): the CTAs in flight
        # read the same query heads' Q / dO and reduce into the same dQ rows
        t_idx = np.tile(order, n_kv_heads)
        heads = np.repeat(np.arange(n_kv_heads), n_tiles)
    else:
        t_idx = np.repeat(order, n_kv_heads)
        heads = np.tile(np.arange(n_kv_heads), n_tiles)
    for name in ("kv_row0", "kv_pos0", "kv_len", "qseg_begin", "qseg_count"):
        items[name] = tiles[name][t_idx]
    items["kv_head"] = heads
    items["flags"] = flags
    return BwdWorkList(items, qsegs, pairs, int(tiles["cost"].sum()) * n_kv_heads)
