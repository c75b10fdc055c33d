import sys, time, math, torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import ops
from paper_2509_21841_b200.worklist import build_worklist
# seed-0 github-like 64K batch stand-in: a few long sequences
import os
from paper_2509_21841_b200 import workloads as W
c2 = [n for _, n in W.c2_batch("github", 0).sequences]
for seqlens in ([65536], [32768, 16384, 8192, 8192], [4096]*16, c2):
    t = sum(seqlens)
    q = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
    k = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
    v = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
    wl = build_worklist(ops.local_fragments(seqlens), 16)
    items, segs = ops.upload_worklist(wl, q.device)
    o = torch.empty_like(q); lse = torch.empty(32, t, device='cuda')
    for _ in range(3): ops.attn_fwd(q, k, v, items, wl.n_items, segs, o, lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    n = 10
    for _ in range(n): ops.attn_fwd(q, k, v, items, wl.n_items, segs, o, lse)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flops = 4 * 128 * 32 * wl.pairs_per_head
    print(f"seqlens={seqlens[:4]} items={wl.n_items} ms={ms:.3f} TFLOP/s={flops/ms/1e9:.1f} ({flops/ms/1e9/1680.9*100:.1f}% of measured)", flush=True)
