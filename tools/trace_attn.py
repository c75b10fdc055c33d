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
buf = (ctypes.c_ulonglong * 8192)()
assert _native.lib().zp_debug_trace(buf, 8192) == 0
A = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
med = lambda x: float(np.median(x))
for cta in (0, 1):
    a = A[cta * 4096:(cta + 1) * 4096]
    sm = [a[tt * 1280: tt * 1280 + 1280].reshape(256, 5) for tt in range(2)]
    n = int((sm[0][:, 0] > 0).sum())
    if n == 0:
        continue
    lo, hi = 8, min(n, 199)
    print(f"CTA {cta}: tiles traced {n}; stats over tiles {lo}..{hi}")
    for tt in range(2):
        s = sm[tt][lo:hi]
        d = np.diff(s, axis=1)
        print(f"  softmax t={tt}: ld S {med(d[:,0]):.0f}  half0(+max) {med(d[:,1]+d[:,2]):.0f}  half1 {med(d[:,3]):.0f}"
              f"  | period {med(np.diff(s[:,0])):.0f}  half1 arrive -> next S_FULL {med(s[1:,0]-s[:-1,4]):.0f}")
    if cta != 0:
        continue
    m = a[2560:2560 + 1200].reshape(200, 6)[lo:hi]
    print(f"  mma period {med(np.diff(m[:,2])):.0f}")
    for tt in range(2):
        s = sm[tt][lo:hi]
        print(f"  t={tt}: own half0 arrive -> issuer wakes {med(m[:,3*tt]-s[:,2]):.0f}"
              f"  own half1 arrive -> issuer wakes {med(m[:,3*tt+1]-s[:,4]):.0f}"
              f"  wake h1 -> S(next) issued {med(m[1:,3*tt+2]-m[:-1,3*tt+1]):.0f}"
              f"  S issued -> S_FULL seen {med(s[:,0]-m[:,3*tt+2]):.0f}")
# event timeline of CTA 0 for a few consecutive tiles (cycles relative to S0 issue of the first)
a = A[:4096]
sm = [a[tt * 1280: tt * 1280 + 1280].reshape(256, 5) for tt in range(2)]
m = a[2560:2560 + 1200].reshape(200, 6)
ev = []
import os
g0 = 100
if os.environ.get("BOUNDARY"):
    per_ = np.diff(m[:199, 2])
    g0 = int(np.argmax(per_[20:]) + 20) - 1  # the tile before the slowest S0 issue gap
G = range(g0, g0 + 4)
for g in G:
    for tt in range(2):
        ev += [(m[g, 3*tt+2], f"S{tt}({g}) issued"), (sm[tt][g, 0], f"  S{tt}({g}) FULL seen by softmax{tt}"),
               (sm[tt][g, 2], f"  P{tt}({g}) h0 arrive"), (sm[tt][g, 4], f"  P{tt}({g}) h1 arrive"),
               (m[g, 3*tt], f"issuer wakes P{tt}({g}) h0 -> PV h0"), (m[g, 3*tt+1], f"issuer wakes P{tt}({g}) h1 -> PV h1")]
off = int(A[4096 + 4095]) - int(A[4095])  # peer clock - leader clock at the cluster sync
sm1 = [A[4096 + tt * 1280: 4096 + tt * 1280 + 1280].reshape(256, 5) - off for tt in range(2)]
for g in G:
    for tt in range(2):
        ev += [(sm1[tt][g, 0], f"  [peer] S{tt}({g}) FULL seen"), (sm1[tt][g, 2], f"  [peer] P{tt}({g}) h0 arrive"),
               (sm1[tt][g, 4], f"  [peer] P{tt}({g}) h1 arrive")]
print("peer clock offset", off)
base = m[g0, 2]
for t_, name in sorted(ev):
    print(f"{t_ - base:7d}  {name}")
# mean vs median tile period (item boundaries show up in the mean)
per = np.diff(A[2560:2560 + 1200].reshape(200, 6)[8:199, 2])
it_ = A[3760:3760 + 41 * 8].reshape(41, 2, 4)
ok_ = (it_[:-1, 0, 0] > 0) & (it_[:-1, 0, 2] > 0) & (it_[1:, 0, 3] > 0)
e_ = it_[:-1, 0][ok_]
print("item boundary (head 0), cycles: epilogue", np.median(e_[:, 1] - e_[:, 0]),
      " epilogue end -> next item claimed", np.median(e_[:, 2] - e_[:, 1]),
      " claimed -> tiles counted", np.median(it_[1:, 0, 3][ok_] - e_[:, 2]))
print(f"S0 issue period: median {np.median(per):.0f} mean {per.mean():.0f}; slowest 10: {np.sort(per)[-10:]}")
