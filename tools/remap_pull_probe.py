"""Single-process 2-GPU probe of the fused remap pull kernel (ncu target).

GPU 0 pulls ROWS rows of 8 KiB (hidden 4096 bf16) straight out of a buffer on
GPU 1 over NVLink through zp_remap_pull (world=2, my_rank=0).  The handshake is
satisfied in advance (rank 1's "ready" pre-published in rank 0's flag block, no
readers to wait for), so the call runs alone — safe under ncu's kernel
serialisation.  Prints GB/s from CUDA events."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from cuda.bindings import runtime as cudart  # noqa: E402

from paper_2509_21841_b200 import _native  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
row_bytes = 8192
assert torch.cuda.device_count() >= 2
cudart.cudaSetDevice(0)
err, = cudart.cudaDeviceEnablePeerAccess(1, 0)[:1]
src = torch.randn(rows, row_bytes // 2, device="cuda:1", dtype=torch.bfloat16)
dst = torch.empty(rows, row_bytes // 2, device="cuda:0", dtype=torch.bfloat16)
dev = torch.device("cuda", 0)
world = 2
flags = torch.zeros(2 * world, dtype=torch.int32, device=dev)        # rank 0's flag block
flags_peer = torch.zeros(2 * world, dtype=torch.int32, device=dev)   # stands in for rank 1's block
flags[world + 1] = 1 << 30                                             # rank 1: "my rows are final"
i64 = lambda xs: torch.tensor(xs, dtype=torch.int64, device=dev)      # noqa: E731
i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)      # noqa: E731
src_ptrs = i64([0, src.data_ptr()])
flags_ptrs = i64([flags.data_ptr(), flags_peer.data_ptr()])
src_row0, dst_row0, count, readers = i32([0, 0]), i32([0, 0]), i32([0, rows]), i32([0, 0])
lib = _native.lib()
stream = torch.cuda.current_stream(dev)


def call(epoch):
    rc = lib.zp_remap_pull(ctypes.c_void_p(dst.data_ptr()), ctypes.c_int64(row_bytes),
                           ctypes.c_void_p(src_ptrs.data_ptr()), ctypes.c_void_p(src_row0.data_ptr()),
                           ctypes.c_void_p(dst_row0.data_ptr()), ctypes.c_void_p(count.data_ptr()),
                           ctypes.c_void_p(flags_ptrs.data_ptr()), ctypes.c_void_p(readers.data_ptr()),
                           2, 0, epoch, rows, ctypes.c_void_p(stream.cuda_stream))
    assert rc == 0, rc


with torch.cuda.device(0):
    call(1)
    torch.cuda.synchronize(0)
    assert torch.equal(dst.cpu(), src.cpu()), "pulled rows differ"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(iters):
        call(2 + it)
    e1.record()
    torch.cuda.synchronize(0)
    ms = e0.elapsed_time(e1) / iters
print(f"remap pull 1->0: {rows} rows x {row_bytes} B = {rows * row_bytes / 1e9:.2f} GB in {ms:.3f} ms "
      f"-> {rows * row_bytes / ms / 1e6:.1f} GB/s ({rows * row_bytes / ms / 1e6 / 900 * 100:.1f}% of 900)")
