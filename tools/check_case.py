"""Error of one varlen attention case against the fp32 reference (debug aid)."""
import sys
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_2509_21841_b200 import ops
from test_gpu_attention import make_qkv, ref_attention  # noqa
seqlens = [int(x) for x in sys.argv[2:]] or [3000, 700]
qscale = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
t = sum(seqlens)
q, k, v = make_qkv(t, seed=len(seqlens))
q = (q.float() * qscale).to(torch.bfloat16)
o, lse = ops.varlen_attention(q, k, v, seqlens)
torch.cuda.synchronize()
r = 0
for n in seqlens:
    pos = torch.arange(n, device="cuda")
    ro, rl = ref_attention(q[r:r + n], k[r:r + n], v[r:r + n], pos, pos)
    e = (o[r:r + n].float() - ro).abs()
    rows = e.amax(dim=2).amax(dim=1)
    bad = (rows > 2e-2).nonzero().flatten()
    print(f"seq len {n}: max err {e.max().item():.4f}, lse err {(lse[:, r:r + n] - rl).abs().max().item():.4f}, "
          f"bad rows {bad.numel()} first {bad[:10].tolist()}")
    r += n
