"""Where the end-to-end (host-buffer) step time goes on one B200."""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_2509_21841_b200 import engine, workloads as W

batch = W.c2_batch("github", 0)
cluster = W.cluster_for(batch, 1)
ctx = engine.RankContext(0, 1, torch.device("cuda", 0))
layer = engine.ZeppelinLayer(cluster, ctx)
layer.prepare(batch)
rows = layer.program.rows
hq_ = torch.randn(rows, 32, 128, dtype=torch.bfloat16).pin_memory()
hk_ = torch.randn(rows, 8, 128, dtype=torch.bfloat16).pin_memory()
hv_ = torch.randn(rows, 8, 128, dtype=torch.bfloat16).pin_memory()
ho_ = [torch.empty(rows, 32, 128, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
dq = torch.empty(rows, 32, 128, dtype=torch.bfloat16, device="cuda")
dk = torch.empty(rows, 8, 128, dtype=torch.bfloat16, device="cuda")


def timed(fn, n=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3 / n


print("H2D q+k+v ms", timed(lambda: (dq.copy_(hq_, non_blocking=True), dk.copy_(hk_, non_blocking=True),
                                      dk.copy_(hv_, non_blocking=True))))
print("D2H o ms", timed(lambda: ho_[0].copy_(dq, non_blocking=True)))
print("prepare ms", timed(lambda: layer.prepare(batch)))
i = [0]


def step(prep):
    if prep:
        layer.prepare(batch)
    layer.step_host(hq_, hk_, hv_, ho_[i[0] % 2])
    i[0] += 1


print("step_host (no prepare) ms", timed(lambda: step(False)))
print("step_host (+prepare) ms", timed(lambda: step(True)))
q = torch.randn(rows, 32, 128, dtype=torch.bfloat16, device="cuda")
k = torch.randn(rows, 8, 128, dtype=torch.bfloat16, device="cuda")
v = torch.randn(rows, 8, 128, dtype=torch.bfloat16, device="cuda")
print("device-only forward ms", timed(lambda: layer.forward(q, k, v)))
