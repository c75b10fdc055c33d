"""Attention backward (zp_attn_bwd) against a plain PyTorch
fp32 autograd reference of the same causal GQA attention.

Tolerance: bf16 inputs, P and dS rounded to bf16 before the tensor-core
products (as every flash backward does), fp32 accumulation; we require
max|err| <= 2e-2 * max|ref| per gradient (plus 2e-3 absolute slack)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_REL, TOL_ABS = 2e-2, 2e-3


def _ref_grads(q, k, v, dout, seqlens):
    hq, hkv = q.shape[1], k.shape[1]
    qf, kf, vf = (t.float().detach().requires_grad_(True) for t in (q, k, v))
    outs = []
    r = 0
    for n in seqlens:
        if n == 0:
            continue
        qs = qf[r:r + n].transpose(0, 1)
        ks = kf[r:r + n].repeat_interleave(hq // hkv, dim=1).transpose(0, 1)
        vs = vf[r:r + n].repeat_interleave(hq // hkv, dim=1).transpose(0, 1)
        outs.append(torch.nn.functional.scaled_dot_product_attention(qs, ks, vs, is_causal=True).transpose(0, 1))
        r += n
    o = torch.cat(outs)
    o.backward(dout.float())
    return qf.grad, kf.grad, vf.grad


def _check(name, got, ref):
    err = (got.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= TOL_REL * scale + TOL_ABS, f"{name}: max err {err:.3e} vs max |ref| {scale:.3e}"


@pytest.mark.parametrize("seqlens,hq,hkv,qscale", [
    ([1000], 32, 8, 1.0),
    ([300, 17, 129, 64, 1, 200], 32, 8, 1.0),
    ([2048, 511], 16, 8, 1.0),
    ([777], 4, 2, 1.0),
    ([0, 200, 0, 65], 32, 8, 1.0),
    ([1500], 32, 8, 4.0),
])
def test_local_backward_matches_fp32_autograd(seqlens, hq, hkv, qscale):
    from paper_2509_21841_b200 import ops
    t = sum(seqlens)
    g = torch.Generator().manual_seed(7)
    q = (torch.randn(t, hq, 128, generator=g) * qscale).to(torch.bfloat16).cuda()
    k = torch.randn(t, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(t, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    dout = torch.randn(t, hq, 128, generator=g).to(torch.bfloat16).cuda()
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    dq, dk, dv = ops.varlen_attention_backward(q, k, v, o, lse, dout, seqlens)
    torch.cuda.synchronize()
    rq, rk, rv = _ref_grads(q, k, v, dout, seqlens)
    _check("dv", dv, rv)
    _check("dk", dk, rk)
    _check("dq", dq, rq)


def test_backward_is_deterministic_in_dk_dv():
    """dK/dV are written once per key tile (no atomics): bitwise repeatable."""
    from paper_2509_21841_b200 import ops
    seqlens = [1500, 300]
    t = sum(seqlens)
    g = torch.Generator().manual_seed(3)
    q = torch.randn(t, 32, 128, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(t, 8, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(t, 8, 128, generator=g).to(torch.bfloat16).cuda()
    dout = torch.randn(t, 32, 128, generator=g).to(torch.bfloat16).cuda()
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    a = ops.varlen_attention_backward(q, k, v, o, lse, dout, seqlens)
    b = ops.varlen_attention_backward(q, k, v, o, lse, dout, seqlens)
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    assert (a[0].float() - b[0].float()).abs().max().item() <= 1e-2 * a[0].float().abs().max().item()


def _plan_backward_check(plan, seed):
    """Every rank of a plan (rings included) emulated on one GPU: forward,
    then backward with travelling dK/dV; gradients gathered per sequence
    against fp32 autograd of whole-sequence causal attention."""
    from paper_2509_21841_b200 import schedule as S
    from paper_2509_21841_b200.emulate import emulate_backward_on_one_gpu, emulate_ranks_on_one_gpu
    sched = S.build_schedule(plan)
    g = torch.Generator().manual_seed(seed)
    seqs = sorted(plan.sequence_lengths.items())
    mk = lambda h: {s: torch.randn(n, h, 128, generator=g).to(torch.bfloat16) for s, n in seqs}  # noqa: E731
    sq, sk, sv, sdo = mk(32), mk(8), mk(8), mk(32)
    outs = emulate_ranks_on_one_gpu(plan, sched, sq, sk, sv)
    grads = emulate_backward_on_one_gpu(plan, sched, sq, sk, sv, sdo, outs)
    # scatter rank-layout gradients back to sequences
    got = {s: [torch.zeros(n, 32, 128), torch.zeros(n, 8, 128), torch.zeros(n, 8, 128)] for s, n in seqs}
    for r in range(plan.num_ranks):
        at = 0
        for f in plan.fragments[r]:
            for j in range(3):
                got[f.sequence_id][j][f.start:f.end] = grads[r][j][at:at + f.tokens].float().cpu()
            at += f.tokens
    for s, n in seqs:
        rq, rk, rv = _ref_grads(sq[s].cuda(), sk[s].cuda(), sv[s].cuda(), sdo[s].cuda(), [n])
        _check(f"seq {s} dq", got[s][0], rq.cpu())
        _check(f"seq {s} dk", got[s][1], rk.cpu())
        _check(f"seq {s} dv", got[s][2], rv.cpu())


@pytest.mark.parametrize("g,lengths", [
    (2, [3000, 100, 40]),
    (4, [4096, 1000, 33, 600, 129]),
    (8, [5000, 1200, 1100, 300, 64, 1]),
])
def test_ring_backward_matches_fp32_autograd(g, lengths):
    from paper_2509_21841_b200 import plan as P
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import ClusterSpec
    total = sum(lengths)
    cluster = ClusterSpec(1, g, -(-total * 105 // (100 * g)), 1.0, 1.0)
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), cluster)
    assert plan.ring_groups
    _plan_backward_check(plan, seed=g)
