"""CPU interpreter of the kernel's work-item contract (zp_attn_item / zp_kv_seg,
include/zeppelin_b200.h) — test infrastructure.

It executes a work list exactly as documented for ``zp_attn_fwd`` (tile of
<=128 query rows x head pair, KV segments with global positions, causal mask
k_pos <= q_pos, partial-state load/store flags), in float64, so host-side
tables can be validated against ``attention.run_plan`` on a CPU and the GPU
kernel can be validated against the same tables.
"""

from __future__ import annotations

import numpy as np

LOAD, STORE = 1, 2


class State:
    def __init__(self, rows, hq, d):
        self.o = np.zeros((rows, hq, d))
        self.m = np.full((hq, rows), -np.inf)
        self.l = np.zeros((hq, rows))


def run_items(items, segs, q, k, v, o, lse, state, scale):
    """q [Tq,Hq,d], k/v [Tk,Hkv,d] (float64 arrays); o/lse written in place."""
    hq = q.shape[1]
    grp = hq // k.shape[1]
    for it in items:
        r0, p0, n = int(it["q_row0"]), int(it["q_pos0"]), int(it["q_len"])
        qpos = p0 + np.arange(n)
        kr, kp = [], []
        for s in segs[int(it["seg_begin"]): int(it["seg_begin"]) + int(it["seg_count"])]:
            kr.append(int(s["row0"]) + np.arange(int(s["len"])))
            kp.append(int(s["pos0"]) + np.arange(int(s["len"])))
        kr = np.concatenate(kr)
        kp = np.concatenate(kp)
        vis = kp[None, :] <= qpos[:, None]
        for h in (2 * int(it["head_pair"]), 2 * int(it["head_pair"]) + 1):
            sc = q[r0:r0 + n, h, :] @ k[kr, h // grp, :].T * scale
            sc = np.where(vis, sc, -np.inf)
            if it["flags"] & LOAD:
                s0 = int(it["state_row0"])
                m_old = state.m[h, s0:s0 + n]
                l_old = state.l[h, s0:s0 + n]
                o_old = state.o[s0:s0 + n, h, :]
            else:
                m_old = np.full(n, -np.inf)
                l_old = np.zeros(n)
                o_old = np.zeros((n, q.shape[2]))
            m_new = np.maximum(m_old, sc.max(axis=1))
            m_use = np.where(np.isfinite(m_new), m_new, 0.0)
            alpha = np.exp(m_old - m_use)
            p = np.exp(sc - m_use[:, None])
            l_new = l_old * alpha + p.sum(axis=1)
            o_new = o_old * alpha[:, None] + p @ v[kr, h // grp, :]
            if it["flags"] & STORE:
                s0 = int(it["state_row0"])
                state.m[h, s0:s0 + n] = m_new
                state.l[h, s0:s0 + n] = l_new
                state.o[s0:s0 + n, h, :] = o_new
            else:
                with np.errstate(invalid="ignore", divide="ignore"):
                    o[r0:r0 + n, h, :] = np.where(l_new[:, None] > 0, o_new / l_new[:, None], 0.0)
                    lse[h, r0:r0 + n] = np.where(l_new > 0, m_use + np.log(l_new), -np.inf)


def run_bwd_items(items, qsegs, q, k, v, dout, lse, delta, scale, qblock=64):
    """Execute backward work items (zp_bwd_item, include/zeppelin_b200.h) in
    float64 exactly as documented: every 128-key tile against the 64-row
    query blocks of its query segments from the first block that can see the
    tile's first key, all query heads of the GQA group, mask k_pos <= q_pos.
    lse [Hq, Tq] (natural log) and delta [Hq, Tq] = rowsum(dO * O) come from
    the forward.  Returns (dq, dk, dv, pairs_per_head) with dk/dv written per item (the
    ACCUMULATE flag adds)."""
    hq, d = q.shape[1], q.shape[2]
    hkv = k.shape[1]
    grp = hq // hkv
    dq = np.zeros(q.shape)
    dk = np.zeros(k.shape)
    dv = np.zeros(k.shape)
    pairs = 0
    for it in items:
        kr0, kp0, kn, g = (int(it[x]) for x in ("kv_row0", "kv_pos0", "kv_len", "kv_head"))
        kpos = kp0 + np.arange(kn)
        gk = np.zeros((kn, d))
        gv = np.zeros((kn, d))
        for s in qsegs[int(it["qseg_begin"]): int(it["qseg_begin"]) + int(it["qseg_count"])]:
            r0, p0, n = int(s["row0"]), int(s["pos0"]), int(s["len"])
            if n <= 0 or p0 + n - 1 < kp0:
                continue
            b0 = max(0, (kp0 - p0) // qblock) if kp0 > p0 else 0
            rows = np.arange(b0 * qblock, n)
            qpos = p0 + rows
            vis = kpos[None, :] <= qpos[:, None]
            if g == 0:
                pairs += int(vis.sum())
            for h in range(g * grp, (g + 1) * grp):
                qq = q[r0 + rows, h, :]
                kk = k[kr0:kr0 + kn, g, :]
                vv = v[kr0:kr0 + kn, g, :]
                do = dout[r0 + rows, h, :]
                p = np.where(vis, np.exp(qq @ kk.T * scale - lse[h, r0 + rows][:, None]), 0.0)
                dp = do @ vv.T
                ds = p * (dp - delta[h, r0 + rows][:, None])
                gv += p.T @ do
                gk += ds.T @ qq * scale
                dq[r0 + rows, h, :] += ds @ kk * scale
        acc = int(it["flags"]) & 1
        if acc:
            dk[kr0:kr0 + kn, g] += gk
            dv[kr0:kr0 + kn, g] += gv
        else:
            dk[kr0:kr0 + kn, g] = gk
            dv[kr0:kr0 + kn, g] = gv
    return dq, dk, dv, pairs
