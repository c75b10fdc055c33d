"""Attention backward at the benchmarked size (the batch
of BASELINE.json config 2 that `bench.py --workload train` times): the whole
64K-token github batch (longest sequence 50,654 tokens) through the
production backward kernel, against a chunked fp32 GPU backward
(tests/fp32_reference.py) that is itself checked against torch autograd.

Contract (the one tests/test_gpu_backward.py uses at small sizes): per
gradient, max |got - ref| <= 2e-2 * max |ref| + 2e-3; mean-rel
(sum |got - ref| / sum |ref|) is reported beside it.  The kernel's inputs are
its own forward's bf16 O and LSE (what a training step feeds it); the
reference recomputes O and LSE in fp32."""

import json
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

from fp32_reference import causal_attention_backward_fp32
from test_gpu_backward import TOL_ABS, TOL_REL, _ref_grads

from paper_2509_21841_b200 import ops, workloads as W


def _record(name: str, payload: dict) -> None:
    path = os.environ.get("ZP_PARITY_JSON")
    print(name, json.dumps(payload))
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"case": name, **payload}) + "\n")


def _inputs(t: int, seed: int, hq: int = 32, hkv: int = 8):
    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda h: torch.randn(t, h, 128, device="cuda", generator=g, dtype=torch.bfloat16)  # noqa: E731
    return mk(hq), mk(hkv), mk(hkv), mk(hq)


def test_chunked_fp32_backward_matches_autograd():
    """The reference itself: chunked fp32 backward == torch autograd (fp32)."""
    seqlens = [700]
    q, k, v, do = _inputs(700, 5)
    rq, rk, rv = _ref_grads(q, k, v, do, seqlens)
    dq, dk, dv = causal_attention_backward_fp32(q, k, v, do, block=128)
    for name, a, b in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        err = (a - b).abs().max().item()
        assert err <= 1e-4 * b.abs().max().item() + 1e-5, (name, err)


def test_backward_full_c2_batch_matches_fp32():
    seqlens = [n for _, n in W.c2_batch("github", 0).sequences]
    assert sum(seqlens) == 65536 and max(seqlens) == 50654
    t = sum(seqlens)
    q, k, v, do = _inputs(t, 11)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    dq, dk, dv = ops.varlen_attention_backward(q, k, v, o, lse, do, seqlens)
    torch.cuda.synchronize()
    stats = {}
    r = 0
    acc = {name: [0.0, 0.0, 0.0, 0.0] for name in ("dq", "dk", "dv")}  # max err, max ref, sum err, sum ref
    for n in seqlens:
        rq, rk, rv = causal_attention_backward_fp32(q[r:r + n], k[r:r + n], v[r:r + n], do[r:r + n])
        for name, got, ref in (("dq", dq[r:r + n], rq), ("dk", dk[r:r + n], rk), ("dv", dv[r:r + n], rv)):
            d = (got.float() - ref).abs()
            a = acc[name]
            a[0] = max(a[0], d.max().item())
            a[1] = max(a[1], ref.abs().max().item())
            a[2] += d.double().sum().item()
            a[3] += ref.double().abs().sum().item()
        del rq, rk, rv
        r += n
    for name, (emax, rmax, esum, rsum) in acc.items():
        stats[name] = {"max_abs": emax, "max_ref": rmax, "mean_rel": esum / rsum}
    _record("backward_c2_github_seed0", stats)
    for name, st in stats.items():
        assert st["max_abs"] <= TOL_REL * st["max_ref"] + TOL_ABS, (name, st)


@pytest.mark.parametrize("gpus", [2, 4, 8])
def test_ring_backward_c3_matches_fp32(gpus):
    """Config 3 at G=2/4/8 (the 131,072-token sequence in a ring; at G=8 five
    rings): every rank emulated on one GPU through the production forward
    and backward executors (ring rounds, KV hops, travelling dK/dV totals),
    gradients gathered per sequence against the chunked fp32 backward."""
    from paper_2509_21841_b200 import plan as P, schedule as S
    from paper_2509_21841_b200.emulate import emulate_backward_on_one_gpu, emulate_ranks_on_one_gpu
    batch = W.c3_batch(gpus)
    plan = P.build_plan(batch, W.cluster_for(batch, gpus))
    assert plan.ring_groups
    sched = S.build_schedule(plan)
    seqs = sorted(plan.sequence_lengths.items())
    g = torch.Generator().manual_seed(21)
    mk = lambda h: {s: torch.randn(n, h, 128, generator=g).to(torch.bfloat16) for s, n in seqs}  # noqa: E731
    sq, sk, sv, sdo = mk(32), mk(8), mk(8), mk(32)
    outs = emulate_ranks_on_one_gpu(plan, sched, sq, sk, sv)
    grads = emulate_backward_on_one_gpu(plan, sched, sq, sk, sv, sdo, outs)
    got = {s: [torch.zeros(n, 32, 128), torch.zeros(n, 8, 128), torch.zeros(n, 8, 128)] for s, n in seqs}
    for r in range(plan.num_ranks):
        at = 0
        for f in plan.fragments[r]:
            for j in range(3):
                got[f.sequence_id][j][f.start:f.end] = grads[r][j][at:at + f.tokens].float().cpu()
            at += f.tokens
    acc = {name: [0.0, 0.0, 0.0, 0.0] for name in ("dq", "dk", "dv")}
    for s, n in seqs:
        ref = causal_attention_backward_fp32(sq[s].cuda(), sk[s].cuda(), sv[s].cuda(), sdo[s].cuda())
        for j, name in enumerate(("dq", "dk", "dv")):
            d = (got[s][j].cuda() - ref[j]).abs()
            a = acc[name]
            a[0] = max(a[0], d.max().item())
            a[1] = max(a[1], ref[j].abs().max().item())
            a[2] += d.double().sum().item()
            a[3] += ref[j].double().abs().sum().item()
        del ref
    stats = {name: {"max_abs": e, "max_ref": m, "mean_rel": es / rs} for name, (e, m, es, rs) in acc.items()}
    _record(f"ring_backward_c3_g{gpus}", stats)
    for name, st in stats.items():
        assert st["max_abs"] <= TOL_REL * st["max_ref"] + TOL_ABS, (name, st)
