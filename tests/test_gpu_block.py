"""Config 5 building blocks on a B200: the block's elementwise kernels against
torch fp32, and one full Llama-3-8B block (world 1) against the plain PyTorch
fp32 reference block (tolerances written per check)."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2509_21841_b200 import block as B, ops, single_box
from paper_2509_21841_b200.batch import SequenceBatch
from paper_2509_21841_b200.engine import RankContext


def test_rmsnorm_matches_fp32():
    x = torch.randn(333, 4096, device="cuda").to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(4096, device="cuda")).to(torch.bfloat16)
    y = ops.rmsnorm(x, w, 1e-5).float()
    xf = x.float()
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert (y - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


def test_swiglu_matches_fp32():
    gu = torch.randn(257, 2 * 14336, device="cuda").to(torch.bfloat16)
    a = ops.swiglu(gu).float()
    g, u = gu.float()[:, :14336], gu.float()[:, 14336:]
    ref = torch.nn.functional.silu(g) * u
    assert (a - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-3


def test_rope_split_matches_fp32():
    rows, hq, hkv = 300, 32, 8
    qkv = torch.randn(rows, (hq + 2 * hkv) * 128, device="cuda").to(torch.bfloat16)
    pos = torch.randint(0, 131072, (rows,), device="cuda", dtype=torch.int32)
    cos, sin = B.rope_tables(131072, "cuda")
    q, k, v = ops.rope_split(qkv, pos, cos, sin, hq, hkv)
    inv = B.ROPE_THETA ** (-torch.arange(0, 128, 2, dtype=torch.float64, device="cuda") / 128)
    ang = pos.double()[:, None] * inv[None]
    c, s = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    f = qkv.float()

    def rot(t):
        return torch.cat([t[..., :64] * c - t[..., 64:] * s, t[..., 64:] * c + t[..., :64] * s], -1)

    rq = rot(f[:, :hq * 128].view(rows, hq, 128))
    rk = rot(f[:, hq * 128:(hq + hkv) * 128].view(rows, hkv, 128))
    assert (q.float() - rq).abs().max().item() <= 3e-2
    assert (k.float() - rk).abs().max().item() <= 3e-2
    assert torch.equal(v.view(rows, -1), qkv[:, (hq + hkv) * 128:])


def test_full_block_single_gpu_matches_fp32_reference():
    lengths = [900, 260, 1300, 37]
    batch = SequenceBatch(tuple(enumerate(lengths)))
    cluster = single_box(1, batch.total_tokens)
    w = B.BlockWeights.random("cuda", seed=3)
    blk = B.ZeppelinBlock(cluster, w, RankContext(0, 1), max_pos=4096)
    blk.prepare(batch)
    g = torch.Generator(device="cuda").manual_seed(5)
    x_seq = {s: torch.randn(n, 4096, device="cuda", generator=g).to(torch.bfloat16) for s, n in enumerate(lengths)}
    toks = B.linear_tokens(blk.plan, blk.layout, 0)
    x = torch.stack([x_seq[int(s)][int(p)] for s, p in toks])
    out = blk.forward(x)
    torch.cuda.synchronize()
    ref = B.reference_block(x_seq, w)
    want = torch.stack([ref[int(s)][int(p)] for s, p in toks])
    err = (out.float() - want).abs()
    scale = want.abs().max().item()
    # bf16 activations between every op; K = 4096 / 14336 GEMMs
    assert err.max().item() <= 3e-2 * scale, (err.max().item(), scale)
    assert err.mean().item() <= 3e-3 * scale, (err.mean().item(), scale)
