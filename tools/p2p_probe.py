"""Calibrate NVLink peer copies on 2 GPUs, wall-clock timed after full syncs."""
import time

import torch

n = 1 << 30
a0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
b1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
a1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
b0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")


def sync():
    torch.cuda.synchronize("cuda:0")
    torch.cuda.synchronize("cuda:1")


for label, fn in [
    ("push 0->1 on dev0 stream", lambda: b1.copy_(a0, non_blocking=True)),
]:
    with torch.cuda.device(0):
        for _ in range(3):
            fn()
        sync()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        sync()
        dt = (time.perf_counter() - t0) / 20
    print(f"{label}: {n / dt / 1e9:.1f} GB/s")
s1 = torch.cuda.Stream("cuda:1")
with torch.cuda.device(0):
    for _ in range(3):
        b1.copy_(a0, non_blocking=True)
    sync()
    t0 = time.perf_counter()
    for _ in range(20):
        b1.copy_(a0, non_blocking=True)
        with torch.cuda.device(1), torch.cuda.stream(s1):
            b0.copy_(a1, non_blocking=True)
    sync()
    dt = (time.perf_counter() - t0) / 20
print(f"bidirectional: {n / dt / 1e9:.1f} GB/s per direction")
