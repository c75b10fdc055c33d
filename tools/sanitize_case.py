"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck):
forward (pair + single + parity + ring-resume), backward, copy_rows, the
emulated fused remap and the copy-engine ring hop.
  compute-sanitizer --tool memcheck python tools/sanitize_case.py [fwd|bwd|move]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_21841_b200 import ops  # noqa: E402


def fwd():
    for hq, hkv, seqlens in ((32, 8, [300, 129, 1]), (16, 8, [257, 64])):
        t = sum(seqlens)
        q = torch.randn(t, hq, 128, device="cuda", dtype=torch.bfloat16)
        k = torch.randn(t, hkv, 128, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(t, hkv, 128, device="cuda", dtype=torch.bfloat16)
        ops.varlen_attention(q, k, v, seqlens)
        ops.varlen_attention(q, k, v.to(torch.float16), seqlens)
    from paper_2509_21841_b200 import plan as P, schedule as S, workloads as W
    from paper_2509_21841_b200.emulate import emulate_ranks_on_one_gpu
    plan = P.build_plan(W.c1_batch(), W.c1_cluster())
    sched = S.build_schedule(plan)
    seqs = sorted(plan.sequence_lengths.items())
    mk = lambda n, h: torch.randn(n, h, 128).to(torch.bfloat16)  # noqa: E731
    emulate_ranks_on_one_gpu(plan, sched, {s: mk(n, 32) for s, n in seqs}, {s: mk(n, 8) for s, n in seqs},
                             {s: mk(n, 8) for s, n in seqs})
    torch.cuda.synchronize()


def bwd():
    seqlens = [300, 129, 1]
    t = sum(seqlens)
    q = torch.randn(t, 32, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(t, 8, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(t, 8, 128, device="cuda", dtype=torch.bfloat16)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    ops.varlen_attention_backward(q, k, v, o, lse, torch.randn_like(q), seqlens)
    torch.cuda.synchronize()


def move():
    from paper_2509_21841_b200.emulate import emulate_remap_on_one_gpu
    from paper_2509_21841_b200.remap import remap_layout
    lay = remap_layout([700, 10, 300])
    xs = [torch.randn(n, 512, device="cuda").to(torch.bfloat16) for n in lay.attn_rows]
    for method in ("pull", "push"):
        ys = emulate_remap_on_one_gpu(lay, xs, method)
        emulate_remap_on_one_gpu(lay, ys, method, inverse=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    {"fwd": fwd, "bwd": bwd, "move": move}[sys.argv[1] if len(sys.argv) > 1 else "fwd"]()
    print("case done")
