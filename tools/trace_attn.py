"""Per-stage SM-clock breakdown of the attention pipeline (diagnostic build).

Run with ZP_LIB_PATH pointing at a library built with -DZP_TRACE; prints, for
CTA 0, the median cycles of each softmax stage and of the MMA-issue gaps."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import ops, _native
from paper_2509_21841_b200.worklist import build_worklist

seqlens = [int(x) for x in (sys.argv[1:] or ['65536'])]
t = sum(seqlens)
q = torch.randn(t, 32, 128, device='cuda', dtype=torch.bfloat16)
k = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
v = torch.randn(t, 8, 128, device='cuda', dtype=torch.bfloat16)
wl = build_worklist(ops.local_fragments(seqlens), 16)
items, segs = ops.upload_worklist(wl, q.device)
o = torch.empty_like(q); lse = torch.empty(32, t, device='cuda')
for _ in range(2):
    ops.attn_fwd(q, k, v, items, wl.n_items, segs, o, lse)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
assert _native.lib().zp_debug_trace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
sm = [a[tt * 1280: tt * 1280 + 1280].reshape(256, 5) for tt in range(2)]
mm = a[2560:2560 + 1024].reshape(256, 4)
n = int((sm[0][:, 0] > 0).sum())
lo, hi = 8, min(n, 200)
print(f"tiles traced: {n}; stats over tiles {lo}..{hi}")
for tt in range(2):
    s = sm[tt][lo:hi]
    d = np.diff(s, axis=1)
    print(f"softmax t={tt}: ld S {np.median(d[:,0]):.0f}  max {np.median(d[:,1]):.0f}  exp+stP {np.median(d[:,2]):.0f}"
          f"  wait/fence/arrive {np.median(d[:,3]):.0f}  | S_FULL->S_FULL period {np.median(np.diff(s[:,0])):.0f}"
          f"  arrive->next S_FULL {np.median(s[1:,0]-s[:-1,4]):.0f}")
m = mm[lo:hi]
print(f"mma: P0 wait->S0 issued {np.median(m[:,1]-m[:,0]):.0f}  P1 wait->S1 issued {np.median(m[:,3]-m[:,2]):.0f}"
      f"  period {np.median(np.diff(m[:,0])):.0f}")
# cross-role latencies: softmax arrive (t) -> MMA sees P_FULL(t) for the same tile
for tt in range(2):
    lat = m[1:, 2 * tt] - sm[tt][lo:hi - 1, 4]
    print(f"t={tt}: softmax arrive -> MMA wakes {np.median(lat):.0f};  MMA S issued -> softmax S_FULL {np.median(sm[tt][lo+1:hi,0] - m[:-1, 2*tt+1]):.0f}")
