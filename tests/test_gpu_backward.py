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


@pytest.mark.parametrize("seqlens,hq,hkv", [
    ([1000], 32, 8),
    ([300, 17, 129, 64, 1, 200], 32, 8),
    ([2048, 511], 16, 8),
    ([777], 4, 2),
])
def test_local_backward_matches_fp32_autograd(seqlens, hq, hkv):
    from paper_2509_21841_b200 import ops
    t = sum(seqlens)
    g = torch.Generator().manual_seed(7)
    q = torch.randn(t, hq, 128, generator=g).to(torch.bfloat16).cuda()
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
