"""Stream-flag probe (zp_stream_wait_flag / zp_stream_write_flag / zp_ring_hop)
on one GPU: stream A waits for a flag that stream B writes after a delay
kernel, then copies; checks ordering and prints timings.  Run under
`timeout` — a broken wait hangs."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_21841_b200 import _native  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    a, b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    flags = torch.zeros(8, dtype=torch.int32, device=dev)
    src = torch.arange(1 << 20, dtype=torch.int32, device=dev)
    dst = torch.zeros_like(src)
    # warm every kernel used below so no module is loaded while a wait is pending
    with torch.cuda.stream(b):
        torch.cuda._sleep(1000)
        src.add_(0)
    torch.cuda.synchronize()
    t0 = time.time()
    # A: wait flag[0] >= 5, then copy src -> dst, then write flag[1] = 7
    _native.call("zp_ring_hop", dst.data_ptr(), src.data_ptr(), src.numel() * 4, flags.data_ptr(), 5, None, 0,
                 flags.data_ptr() + 4, 7, None, 0, int(a.cuda_stream))
    print("enqueued hop", time.time() - t0, flush=True)
    with torch.cuda.stream(b):
        torch.cuda._sleep(200_000_000)  # ~0.1 s of spinning before the write
        print("enqueued sleep", time.time() - t0, flush=True)
        src.add_(1)                      # the hop must see this (write ordered before the flag)
        print("enqueued add", time.time() - t0, flush=True)
    _native.call("zp_stream_write_flag", flags.data_ptr(), 5, int(b.cuda_stream))
    print("enqueued write", time.time() - t0, flush=True)
    _native.call("zp_stream_wait_flag", flags.data_ptr() + 4, 7, int(b.cuda_stream))
    b.synchronize()
    print("b done", time.time() - t0, flush=True)
    a.synchronize()
    print("a done", time.time() - t0, flush=True)
    ok = torch.equal(dst, torch.arange(1 << 20, dtype=torch.int32, device=dev) + 1)
    print("copy saw the write before the flag:", ok, "flags:", flags.tolist())


if __name__ == "__main__":
    main()
