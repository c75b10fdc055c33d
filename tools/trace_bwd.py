"""Stage timing of the backward pipeline (diagnostic ZP_TRACE build), CTA 0."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import ops, _native
from paper_2509_21841_b200.worklist import build_bwd_worklist
t = 65536
q = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
k = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
v = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
do = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
o, lse = ops.varlen_attention(q, k, v, [t])
wl = build_bwd_worklist(ops.local_fragments([t]), 8)
items, qsegs = ops.upload_bwd_worklist(wl, q.device)
delta = torch.empty_like(lse)
dq = torch.zeros(q.shape, dtype=torch.float32, device='cuda')
dk = torch.zeros(k.shape, dtype=torch.float32, device='cuda')
dv = torch.zeros(k.shape, dtype=torch.float32, device='cuda')
ops.attn_bwd_prep(o, do, delta)
ops.attn_bwd(q, k, v, do, lse, delta, dq, dk, dv, items, wl.n_items, qsegs)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
assert _native.lib().zp_debug_btrace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
lo, hi = 8, 200
sm = a[0:1024].reshape(256, 4)[lo:hi]
dqw = a[1024:2048].reshape(256, 4)[lo:hi]
mm = a[2048:3072].reshape(256, 4)[lo:hi]
print(f"softmax: wait SDP {np.median(sm[:,1]-sm[:,0]):.0f}  wait PDS_EMPTY {np.median(sm[:,2]-sm[:,1]):.0f}  compute+arrive {np.median(sm[:,3]-sm[:,2]):.0f}  period {np.median(np.diff(sm[:,3])):.0f}")
print(f"mma: PDS seen -> dQ issued {np.median(mm[:,1]-mm[:,0]):.0f}; softmax arrive -> MMA sees PDS {np.median(mm[:,0]-sm[:,3]):.0f}; period {np.median(np.diff(mm[:,0])):.0f}")
print(f"dq warps: drain+reds {np.median(dqw[:,1]-dqw[:,0]):.0f}; MMA dQ issued -> DQ_FULL seen {np.median(dqw[:,0]-mm[:,1]):.0f}")
print(f"dq warps (warp 8): DQ_FULL -> own box free {np.median(dqw[:,2]-dqw[:,0]):.0f}; -> stores done + reduce issued "
      f"{np.median(dqw[:,1]-dqw[:,2]):.0f}; period {np.median(np.diff(dqw[:,0])):.0f}")
sd = a[3072:4096].reshape(256, 4)[lo:hi]
print(f"issue_sdp(m): wait QDO_FULL {np.median(sd[:,1]-sd[:,0]):.0f}  wait DQ_EMPTY {np.median(sd[:,2]-sd[:,1]):.0f}  issue 16 MMAs {np.median(sd[:,3]-sd[:,2]):.0f}")
print(f"S^T(m) issued -> softmax sees SDP(m) {np.median(sm[:,1]-sd[:,3]):.0f}")
