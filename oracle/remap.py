"""numpy restatement of the remap data movement (rule R3 in SURVEY.md / DESIGN.md).

The reference pins the transfer COUNTS M (remapping.py:187-245); the row rule
is this framework's, fixed once and pinned by tests/golden/remap_permutation.json:
rank i keeps attention rows [0, min(A_i, B_i)) and sends its tail [B_i, A_i)
to receivers j ascending (M[i][j] rows each); receiver j appends blocks in
sender-ascending order.  The inverse replays the moves backwards.
"""

from __future__ import annotations

import numpy as np


def _targets(counts):
    d = len(counts)
    q, r = divmod(int(sum(counts)), d)
    return [q + (i < r) for i in range(d)]


def forward(x_ranks, matrix):
    a = [x.shape[0] for x in x_ranks]
    b = _targets(a)
    m = np.asarray(matrix)
    d = len(a)
    out = []
    for j in range(d):
        parts = [x_ranks[j][:min(a[j], b[j])]]
        for s in range(d):
            if m[s, j]:
                off = b[s] + int(m[s, :j].sum())
                parts.append(x_ranks[s][off:off + int(m[s, j])])
        out.append(np.concatenate(parts, axis=0))
    return out


def inverse(y_ranks, matrix, attn_rows):
    b = [y.shape[0] for y in y_ranks]
    m = np.asarray(matrix)
    d = len(b)
    out = []
    for i in range(d):
        parts = [y_ranks[i][:min(attn_rows[i], b[i])]]
        for j in range(d):
            if m[i, j]:
                off = attn_rows[j] + int(m[:i, j].sum())
                parts.append(y_ranks[j][off:off + int(m[i, j])])
        out.append(np.concatenate(parts, axis=0))
    return out


def source_map(attn_rows, matrix):
    """For every rank's linear-layout row: (source rank, source attention row)."""
    x = [np.stack([np.full(n, r), np.arange(n)], axis=1) for r, n in enumerate(attn_rows)]
    return forward(x, matrix)
