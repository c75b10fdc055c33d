"""Stage timing of the v2 attention pipeline (diagnostic ZP_TRACE build)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import ops, _native
from paper_2509_21841_b200.worklist import build_worklist
t = 65536
q = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
k = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
v = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
wl = build_worklist(ops.local_fragments([t]), 16)
items, segs = ops.upload_worklist(wl, q.device)
o = torch.empty_like(q); lse = torch.empty(32, t, device='cuda')
for _ in range(2):
    ops.attn_fwd(q, k, v, items, wl.n_items, segs, o, lse)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
assert _native.lib().zp_debug_trace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
lo, hi = 8, 200
for tt in range(2):
    s = a[tt * 1280: tt * 1280 + 1280].reshape(256, 5)[lo:hi]
    print(f"softmax t={tt}: wait S {np.median(s[:,1]-s[:,0]):.0f}  ld..max {np.median(s[:,2]-s[:,1]):.0f}"
          f"  exp+arrive {np.median(s[:,3]-s[:,2]):.0f}  period {np.median(np.diff(s[:,1])):.0f}")
m = a[2560:2560 + 1024].reshape(256, 4)[lo:hi]
print(f"mma: P0(g) ready -> S(g+2) issued {np.median(m[2:,1]-m[:-2,0]):.0f}  period {np.median(np.diff(m[:,1])):.0f}")
s0 = a[0:1280].reshape(256, 5)[lo:hi]
print(f"S(g) issued -> softmax t0 sees S(g) {np.median(s0[:,1]-m[:,1]):.0f}; softmax P0(g) arrive -> MMA sees {np.median(m[:,0]-s0[:,3]):.0f}")
