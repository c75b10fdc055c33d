"""numpy restatement of what the reference only counts: causal attention.

* ``causal_attention``: O = softmax(q K^T * scale, mask k_pos <= q_pos) V and
  its natural-log LSE, for one sequence's query rows against key rows given by
  global positions (reference attention_engine.py:113-136 defines the mask).
* ``run_plan``: every rank's attention layout computed the way the plan
  prescribes — LocalTask whole-sequence attention (attention_engine.py:
  260-265) and, for rings, round r at position i against the KV held by
  position (i - r) mod g (attention_engine.py:229-244) merged by LSE, with the
  per-round unmasked pair count returned for comparison with the schedule.
"""

from __future__ import annotations

import numpy as np

BLOCK = 1024


def causal_attention(q, k, v, q_pos, k_pos, scale, dtype=np.float64):
    """q [n, Hq, d], k/v [m, Hkv, d] (GQA: q head h uses kv head h // (Hq/Hkv)).
    Returns (o [n, Hq, d], lse [Hq, n], unmasked pair count)."""
    q = np.asarray(q, dtype=dtype)
    k = np.asarray(k, dtype=dtype)
    v = np.asarray(v, dtype=dtype)
    n, hq, d = q.shape
    hkv = k.shape[1]
    grp = hq // hkv
    o = np.zeros((n, hq, d), dtype=dtype)
    lse = np.full((hq, n), -np.inf, dtype=dtype)
    q_pos = np.asarray(q_pos)
    k_pos = np.asarray(k_pos)
    pairs = 0
    for r0 in range(0, n, BLOCK):
        r1 = min(n, r0 + BLOCK)
        vis = k_pos[None, :] <= q_pos[r0:r1, None]          # [b, m]
        pairs += int(vis.sum())
        if not vis.any():
            continue
        for h in range(hq):
            s = q[r0:r1, h, :] @ k[:, h // grp, :].T * scale  # [b, m]
            s = np.where(vis, s, -np.inf)
            mx = s.max(axis=1, keepdims=True)
            safe = np.where(np.isfinite(mx), mx, 0.0)
            p = np.exp(s - safe)
            l = p.sum(axis=1, keepdims=True)
            with np.errstate(invalid="ignore", divide="ignore"):
                o[r0:r1, h, :] = np.where(l > 0, (p @ v[:, h // grp, :]) / np.where(l > 0, l, 1), 0.0)
                lse[h, r0:r1] = np.where(l[:, 0] > 0, safe[:, 0] + np.log(np.where(l[:, 0] > 0, l[:, 0], 1)), -np.inf)
    return o, lse, pairs


def merge(o_a, lse_a, o_b, lse_b):
    """Combine two partial results over disjoint key sets (LSE merge)."""
    m = np.maximum(lse_a, lse_b)
    m = np.where(np.isfinite(m), m, 0.0)
    wa = np.exp(lse_a - m)
    wb = np.exp(lse_b - m)
    tot = wa + wb
    with np.errstate(invalid="ignore", divide="ignore"):
        lse = np.where(tot > 0, m + np.log(np.where(tot > 0, tot, 1)), -np.inf)
        fa = np.where(tot > 0, wa / np.where(tot > 0, tot, 1), 0.0).T[:, :, None]
        fb = np.where(tot > 0, wb / np.where(tot > 0, tot, 1), 0.0).T[:, :, None]
    return o_a * fa + o_b * fb, lse


def layout_rows(plan, rank):
    """(sid, start, end, row0) of the rank's fragments in plan order."""
    out, at = [], 0
    for f in plan.fragments[rank]:
        out.append((f.sequence_id, f.start, f.end, at))
        at += f.tokens
    return out


def gather_rank(seq_tensors, plan, rank):
    """Stack per-sequence rows [len, ...] into the rank's attention layout."""
    parts = [seq_tensors[sid][a:b] for sid, a, b, _ in layout_rows(plan, rank)]
    return np.concatenate(parts, axis=0) if parts else None


def run_plan(plan, schedule, seq_q, seq_k, seq_v, scale, dtype=np.float64):
    """Execute the plan on the CPU.  seq_* map sequence id -> [len, H, d].
    Returns per-rank (o, lse) in attention layout and the unmasked pair count
    of every (ring index, position, round) for comparison with compute_pairs."""
    zone = plan.zone_of
    results = []
    rows_of = [dict(((sid, a), (row0, b - a)) for sid, a, b, row0 in layout_rows(plan, r))
               for r in range(plan.num_ranks)]
    for rank in range(plan.num_ranks):
        n = sum(f.tokens for f in plan.fragments[rank])
        hq, d = next(iter(seq_q.values())).shape[1:]
        results.append((np.zeros((n, hq, d), dtype=dtype), np.full((hq, n), -np.inf, dtype=dtype)))
    in_ring = {s.sequence_id for rs in schedule.rings() for s in rs.ring.sequences}
    for rank in range(plan.num_ranks):
        o, lse = results[rank]
        for f in plan.fragments[rank]:
            if (zone.get(f.sequence_id) == "local" or f.micro_batch > 0) and f.sequence_id not in in_ring:
                row0, n = rows_of[rank][(f.sequence_id, f.start)]
                pos = np.arange(f.start, f.end)
                oo, ll, _ = causal_attention(seq_q[f.sequence_id][f.start:f.end], seq_k[f.sequence_id][f.start:f.end],
                                             seq_v[f.sequence_id][f.start:f.end], pos, pos, scale, dtype)
                o[row0:row0 + n], lse[:, row0:row0 + n] = oo, ll
    round_pairs = {}
    for ri, rs in enumerate(schedule.rings()):
        ring = rs.ring
        g = ring.group_size
        for i, rank in enumerate(ring.members):
            o, lse = results[rank]
            for r in range(g):
                src = (i - r) % g
                cnt = 0
                for s in ring.sequences:
                    kv = s.ranges_by_position[src]
                    if not kv:
                        continue
                    kpos = np.concatenate([np.arange(c, dd) for c, dd in kv])
                    kk = seq_k[s.sequence_id][kpos]
                    vv = seq_v[s.sequence_id][kpos]
                    for a, b in s.ranges_by_position[i]:
                        row0, n = rows_of[rank][(s.sequence_id, a)]
                        oo, ll, p = causal_attention(seq_q[s.sequence_id][a:b], kk, vv, np.arange(a, b), kpos, scale, dtype)
                        cnt += p
                        o[row0:row0 + n], lse[:, row0:row0 + n] = merge(o[row0:row0 + n], lse[:, row0:row0 + n], oo, ll)
                round_pairs[(ri, i, r)] = cnt
    return results, round_pairs
