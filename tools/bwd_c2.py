"""One backward launch on a 64K sequence (ncu target)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import ops
from paper_2509_21841_b200.worklist import build_bwd_worklist
seqlens = [65536]
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
ops.attn_bwd_prep(o, do, delta)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    ops.attn_bwd(q, k, v, do, lse, delta, dq, dk, dv, items, wl.n_items, qsegs)
torch.cuda.synchronize()
print("ok")
