"""Backward A/B on one B200: the fused key-stationary kernel (zp_attn_bwd with
dQ) against two passes (zp_attn_bwd without dQ + the query-stationary
zp_attn_bwd_dq).  Prints TFLOP/s of the 5 useful products for both and the
max difference of their dq / dk / dv."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_21841_b200 import ops  # noqa: E402
from paper_2509_21841_b200.worklist import build_bwd_worklist, build_worklist  # noqa: E402

for seqlens in ([65536], [32768, 16384, 8192, 8192], [4096] * 16):
    t = sum(seqlens)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda h: torch.randn(t, h, 128, device="cuda", generator=g, dtype=torch.bfloat16)  # noqa: E731
    q, k, v, do = mk(32), mk(8), mk(8), mk(32)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    wl = build_bwd_worklist(ops.local_fragments(seqlens), 8)
    items, qsegs = ops.upload_bwd_worklist(wl, q.device)
    qw = build_worklist(ops.local_fragments(seqlens), 32)
    qi, qs = ops.upload_worklist(qw, q.device)
    delta = torch.empty_like(lse)
    ops.attn_bwd_prep(o, do, delta)
    res = {}
    for mode in ("fused", "2pass", "kv_only", "dq_only"):
        dq = torch.zeros(q.shape, dtype=torch.float32, device="cuda")
        dk = torch.zeros(k.shape, dtype=torch.float32, device="cuda")
        dv = torch.zeros(k.shape, dtype=torch.float32, device="cuda")

        def step():
            dq.zero_()
            if mode == "fused":
                ops.attn_bwd(q, k, v, do, lse, delta, dq, dk, dv, items, wl.n_items, qsegs)
            elif mode == "kv_only":
                ops.attn_bwd(q, k, v, do, lse, delta, None, dk, dv, items, wl.n_items, qsegs)
            elif mode == "dq_only":
                ops.attn_bwd_dq(q, k, v, do, lse, delta, dq, qi, qw.n_items, qs)
            else:
                ops.attn_bwd(q, k, v, do, lse, delta, None, dk, dv, items, wl.n_items, qsegs)
                ops.attn_bwd_dq(q, k, v, do, lse, delta, dq, qi, qw.n_items, qs)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n = 5
        e0.record()
        for _ in range(n):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        flops = {"fused": 10, "2pass": 10, "kv_only": 8, "dq_only": 6}[mode] * 128 * 32 * wl.pairs_per_head
        res[mode] = (dq.clone(), dk.clone(), dv.clone())
        print(f"{mode} seqlens={seqlens[:4]} ms={ms:.3f} TFLOP/s={flops / ms / 1e9:.1f}", flush=True)
    diffs = [float((a - b).abs().max()) / max(float(a.abs().max()), 1e-9) for a, b in zip(res["fused"], res["2pass"])]
    # (kv_only: 4 products executed; dq_only: 3 products executed, 1 useful)
    print(f"  rel max diff dq/dk/dv = {diffs}", flush=True)
