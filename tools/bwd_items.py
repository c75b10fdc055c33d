"""Per-item timing of the backward kernel (diagnostic ZP_TRACE build): each
CTA's entry / K,V-landed / exit globaltimer and its step count -> fitted
per-step time and per-item overhead.  usage: tools/bwd_items.py LEN [LEN ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_21841_b200 import _native, ops  # noqa: E402
from paper_2509_21841_b200.worklist import build_bwd_worklist  # noqa: E402

seqlens = [int(x) for x in sys.argv[1:]] or [4096] * 16
t = sum(seqlens)
q = torch.randn(t, 32, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(t, 8, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(t, 8, 128, device="cuda", dtype=torch.bfloat16)
do = torch.randn(t, 32, 128, device="cuda", dtype=torch.bfloat16)
o, lse = ops.varlen_attention(q, k, v, seqlens)
wl = build_bwd_worklist(ops.local_fragments(seqlens), 8)
items, qsegs = ops.upload_bwd_worklist(wl, q.device)
delta = torch.empty_like(lse)
dq = torch.zeros(q.shape, dtype=torch.float32, device="cuda")
dk = torch.zeros(k.shape, dtype=torch.float32, device="cuda")
dv = torch.zeros(k.shape, dtype=torch.float32, device="cuda")
ops.attn_bwd_prep(o, do, delta)
for _ in range(2):
    ops.attn_bwd(q, k, v, do, lse, delta, dq, dk, dv, items, wl.n_items, qsegs)
torch.cuda.synchronize()
lib = _native.lib()
fn = lib.zp_debug_bitems
fn.restype = ctypes.c_int
n = min(wl.n_items, 16384)
buf = (ctypes.c_ulonglong * (n * 4))()
assert fn(buf, n * 4) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(n, 4)
t0 = a[:, 0].min()
dur = (a[:, 2] - a[:, 0]) / 1e3        # us
setup = (a[:, 1] - a[:, 0]) / 1e3      # us until K/V landed
steps = a[:, 3]
A = np.vstack([steps, np.ones_like(steps)]).T
slope, icpt = np.linalg.lstsq(A, dur, rcond=None)[0]
span = (a[:, 2].max() - t0) / 1e3
busy = dur.sum() / 148
print(f"items {n}, steps/item mean {steps.mean():.1f} (min {steps.min()}, max {steps.max()})")
print(f"item duration fit: {slope:.3f} us/step + {icpt:.1f} us/item; median setup (entry -> K,V landed) {np.median(setup):.1f} us")
print(f"kernel span {span:.0f} us, sum of item durations / 148 SMs {busy:.0f} us (fill {busy / span * 100:.0f}%)")
