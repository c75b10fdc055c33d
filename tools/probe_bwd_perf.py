"""Backward attention throughput probe (zp_attn_bwd + prep), one B200."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import ops
from paper_2509_21841_b200.worklist import build_bwd_worklist

for seqlens in ([65536], [32768, 16384, 8192, 8192], [4096] * 16):
    t = sum(seqlens)
    q = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
    k = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
    v = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
    do = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    wl = build_bwd_worklist(ops.local_fragments(seqlens), 8)
    items, qsegs = ops.upload_bwd_worklist(wl, q.device)
    delta = torch.empty_like(lse)
    dq = torch.zeros(q.shape, dtype=torch.float32, device='cuda')
    dk = torch.zeros(k.shape, dtype=torch.float32, device='cuda')
    dv = torch.zeros(k.shape, dtype=torch.float32, device='cuda')

    def step():
        ops.attn_bwd_prep(o, do, delta)
        dq.zero_()
        ops.attn_bwd(q, k, v, do, lse, delta, dq, dk, dv, items, wl.n_items, qsegs)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 5
    e0.record()
    for _ in range(n):
        step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flops = 10 * 128 * 32 * wl.pairs_per_head
    print(f"bwd seqlens={seqlens[:4]} items={wl.n_items} ms={ms:.3f} TFLOP/s={flops/ms/1e9:.1f} "
          f"({flops/ms/1e9/1680.9*100:.1f}% of measured)", flush=True)
