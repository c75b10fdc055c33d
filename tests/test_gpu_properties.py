"""Size-independent properties at BASELINE.json's full sizes (the fp32 / fp64
references only run at small sizes):

* varlen isolation: the config-2 batch (64K tokens, github seed 0) in one
  launch equals each sequence launched alone, bit for bit (masked keys of a
  neighbouring sequence contribute an exact zero);
* backward linearity: dO -> 2 dO doubles dK and dV bit for bit (every
  product and bf16 rounding commutes with a power of two) and dQ up to the
  order of its fp32 atomic reductions."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2509_21841_b200 import ops, workloads as W


def _qkv(t, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda h: torch.randn(t, h, 128, device="cuda", generator=g, dtype=torch.bfloat16)  # noqa: E731
    return mk(32), mk(8), mk(8)


def test_c2_batch_equals_per_sequence_launches():
    seqlens = [n for _, n in W.c2_batch("github", 0).sequences]
    q, k, v = _qkv(sum(seqlens), 0)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    r = 0
    for n in seqlens:
        s = slice(r, r + n)
        o1, l1 = ops.varlen_attention(q[s].contiguous(), k[s].contiguous(), v[s].contiguous(), [n])
        assert torch.equal(o[s], o1), n
        assert torch.equal(lse[:, s], l1), n
        r += n


def _grads(q, k, v, o, lse, dout, seqlens):
    wl = ops.build_bwd_worklist(ops.local_fragments(seqlens), k.shape[1])
    delta = torch.empty_like(lse)
    ops.attn_bwd_prep(o, dout, delta)
    dq = torch.zeros(q.shape, dtype=torch.float32, device="cuda")
    dk = torch.zeros(k.shape, dtype=torch.float32, device="cuda")
    dv = torch.zeros(k.shape, dtype=torch.float32, device="cuda")
    items, qsegs = ops.upload_bwd_worklist(wl, q.device)
    ops.attn_bwd(q, k, v, dout, lse, delta, dq, dk, dv, items, wl.n_items, qsegs)
    return dq, dk, dv


def test_backward_linear_in_dout_at_64k():
    seqlens = [65536]
    q, k, v = _qkv(65536, 1)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    g = torch.Generator(device="cuda").manual_seed(2)
    dout = torch.randn(q.shape, device="cuda", generator=g, dtype=torch.bfloat16)
    dq1, dk1, dv1 = _grads(q, k, v, o, lse, dout, seqlens)
    dq2, dk2, dv2 = _grads(q, k, v, o, lse, dout * 2, seqlens)
    torch.cuda.synchronize()
    assert torch.equal(dk2, 2 * dk1)
    assert torch.equal(dv2, 2 * dv1)
    assert torch.allclose(dq2, 2 * dq1, rtol=1e-5, atol=1e-6 * float(dq1.abs().max()))
