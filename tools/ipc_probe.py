"""Raw copy-engine throughput into a CUDA-IPC mapped peer buffer (no handshake),
2 processes; compare with remap_push_ce to isolate handshake overhead."""
import ctypes
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2509_21841_b200 import engine  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
ctx = engine.RankContext(rank, world, dev)
rows = 131072
peer = engine.PeerBuffer(ctx, rows, 4096)
src = torch.randn(rows, 4096, device=dev).to(torch.bfloat16)
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
for path in ("/usr/local/cuda/lib64/libcudart.so.12", "libcudart.so"):
    try:
        cudart = ctypes.CDLL(path)
        break
    except OSError:
        continue
stream = torch.cuda.current_stream()
dst = int(peer.peer_ptrs[1 - rank].item())
nbytes = rows * 8192
attr = (ctypes.c_int * 16)()
if rank == 0:
    for kind, name in ((3, "D2D"), (4, "Default")):
        for _ in range(3):
            cudart.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src.data_ptr()), ctypes.c_size_t(nbytes), kind, ctypes.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            cudart.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src.data_ptr()), ctypes.c_size_t(nbytes), kind, ctypes.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 10
        print(f"CE memcpy {name} to IPC peer ptr: {nbytes / dt / 1e9:.1f} GB/s", flush=True)
    # peer memcpy with explicit devices
    for _ in range(3):
        cudart.cudaMemcpyPeerAsync(ctypes.c_void_p(dst), 1, ctypes.c_void_p(src.data_ptr()), 0, ctypes.c_size_t(nbytes), ctypes.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        cudart.cudaMemcpyPeerAsync(ctypes.c_void_p(dst), 1, ctypes.c_void_p(src.data_ptr()), 0, ctypes.c_size_t(nbytes), ctypes.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"cudaMemcpyPeerAsync to IPC ptr: {nbytes / dt / 1e9:.1f} GB/s", flush=True)
dist.barrier()
dist.destroy_process_group()
