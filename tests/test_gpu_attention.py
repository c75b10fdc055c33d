"""K1 (local varlen causal attention) and ring-resume parity on a B200.

Reference for this floating-point kernel: plain PyTorch fp32 attention on the
same bf16-rounded inputs (per sequence, GQA expanded), tolerance max-abs 2e-2
on the bf16 output (BASELINE.json north_star)."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2509_21841_b200 import ops
from paper_2509_21841_b200.worklist import QueryFragment, build_worklist, ITEM_LOAD_STATE, ITEM_STORE_STATE

MAX_ABS = 2e-2


def ref_attention(q, k, v, qpos, kpos):
    """fp32 reference: q [n,H,d], k/v [m,Hkv,d], mask kpos <= qpos."""
    hq, hkv = q.shape[1], k.shape[1]
    qf = q.float().transpose(0, 1)
    kf = k.float().repeat_interleave(hq // hkv, dim=1).transpose(0, 1)
    vf = v.float().repeat_interleave(hq // hkv, dim=1).transpose(0, 1)
    s = torch.matmul(qf, kf.transpose(1, 2)) / math.sqrt(q.shape[-1])
    mask = kpos[None, :] <= qpos[:, None]
    s = s.masked_fill(~mask[None], float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    o = torch.matmul(torch.softmax(s, dim=-1), vf).transpose(0, 1)
    return o, lse


def make_qkv(t, hq=32, hkv=8, seed=0):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(t, hq, 128, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(t, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(t, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    return q, k, v


@pytest.mark.parametrize("seqlens,qscale", [([128], 1.0), ([1], 1.0), ([77], 1.0), ([300, 5, 129, 1000], 1.0),
                                            ([2048, 17, 640], 1.0), ([0, 64, 0, 129, 0], 1.0), ([8192], 1.0),
                                            ([3000, 700], 6.0), ([1500], 0.05),
                                            ([100] * 64 + [257] * 8, 1.0)])
def test_varlen_local_matches_fp32(seqlens, qscale):
    """Ragged / empty / long sequences; qscale 6 makes the running max move by
    more than the lazy threshold many times (rescale and speculative-exp
    fallback paths), 0.05 makes the softmax nearly flat; 64 x 100 + 8 x 257 runs
    hundreds of back-to-back one- and three-tile items through the schedule ring
    and the per-head Q barriers."""
    t = sum(seqlens)
    q, k, v = make_qkv(t, seed=len(seqlens))
    q = (q.float() * qscale).to(torch.bfloat16)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    torch.cuda.synchronize()
    r = 0
    for n in seqlens:
        if n == 0:
            continue
        pos = torch.arange(n, device="cuda")
        ro, rl = ref_attention(q[r:r + n], k[r:r + n], v[r:r + n], pos, pos)
        err = (o[r:r + n].float() - ro).abs().max().item()
        assert err <= MAX_ABS, (n, err)
        lerr = (lse[:, r:r + n] - rl).abs().max().item()
        assert lerr <= 1e-2, (n, lerr)
        r += n


def test_resume_state_equals_single_pass():
    """Two launches over two KV segments (ring-round style, with partial
    state) equal one launch over both segments."""
    n = 700
    q, k, v = make_qkv(n, seed=3)
    hq = q.shape[1]
    full = build_worklist([QueryFragment(0, 0, n, [(0, 0, n)])], hq // 2)
    o1 = torch.empty_like(q)
    l1 = torch.empty(hq, n, device="cuda")
    it, sg = ops.upload_worklist(full, q.device)
    ops.attn_fwd(q, k, v, it, full.n_items, sg, o1, l1)
    # split keys [0,300) + [300,700); the second launch resumes
    st_o = torch.zeros(n, hq, 128, device="cuda")
    st_ml = torch.zeros(2, hq, n, device="cuda")
    o2 = torch.empty_like(q)
    l2 = torch.empty(hq, n, device="cuda")
    a = build_worklist([QueryFragment(0, 0, n, [(0, 0, 300)], state_row0=0)], hq // 2,
                       tile_flags=lambda fi, p0, ln: np.full(p0.shape, ITEM_STORE_STATE))
    b = build_worklist([QueryFragment(0, 0, n, [(300, 300, 400)], state_row0=0)], hq // 2,
                       tile_flags=lambda fi, p0, ln: np.full(p0.shape, ITEM_LOAD_STATE))
    it, sg = ops.upload_worklist(a, q.device)
    ops.attn_fwd(q, k, v, it, a.n_items, sg, o2, l2, st_o, st_ml)
    it, sg = ops.upload_worklist(b, q.device)
    ops.attn_fwd(q, k, v, it, b.n_items, sg, o2, l2, st_o, st_ml)
    torch.cuda.synchronize()
    # tiles entirely before key 300 never see segment b (only partials stored)
    rows = slice(256, n)
    assert (o1[rows].float() - o2[rows].float()).abs().max().item() <= 1e-2
    assert (l1[:, rows] - l2[:, rows]).abs().max().item() <= 1e-3


def test_host_fed_pipeline_matches_device_path():
    """ZeppelinLayer.step_host (pinned host inputs, H2D / D2H streams, per-step
    planning with work lists staged through reused pinned slots) over several
    back-to-back steps with DIFFERENT inputs returns exactly what the device
    path computes for each step — no slot is overwritten while in use."""
    from paper_2509_21841_b200 import engine
    from paper_2509_21841_b200.batch import SequenceBatch
    from paper_2509_21841_b200.cluster import single_box
    batch = SequenceBatch(tuple(enumerate([3000, 700, 129, 1])))
    ctx = engine.RankContext(0, 1, torch.device("cuda", 0))
    layer = engine.ZeppelinLayer(single_box(1, batch.total_tokens), ctx)
    layer.prepare(batch)
    rows = layer.program.rows
    steps = 5
    g = torch.Generator().manual_seed(11)
    hq_ = [torch.randn(rows, 32, 128, generator=g).to(torch.bfloat16).pin_memory() for _ in range(steps)]
    hk_ = [torch.randn(rows, 8, 128, generator=g).to(torch.bfloat16).pin_memory() for _ in range(steps)]
    hv_ = [torch.randn(rows, 8, 128, generator=g).to(torch.bfloat16).pin_memory() for _ in range(steps)]
    outs = [torch.empty(rows, 32, 128, dtype=torch.bfloat16).pin_memory() for _ in range(steps)]
    for i in range(steps):
        layer.prepare(batch)
        layer.step_host(hq_[i], hk_[i], hv_[i], outs[i])
    torch.cuda.synchronize()
    for i in range(steps):
        o, _ = layer.attention(hq_[i].cuda(), hk_[i].cuda(), hv_[i].cuda())
        torch.cuda.synchronize()
        assert torch.equal(outs[i], o.cpu()), f"step {i} differs"


def test_pair_contract_violation_fails_loudly():
    """With GQA group 4 the kernel runs CTA pairs; an item list whose pairs do
    not match (here: head pairs swapped) must abort the launch, not return
    wrong numbers.  Run in a child process (a trapped kernel poisons the CUDA
    context)."""
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2509_21841_b200 import ops
from paper_2509_21841_b200.worklist import build_worklist
q = torch.randn(256, 32, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(256, 8, 128, device="cuda", dtype=torch.bfloat16)
wl = build_worklist(ops.local_fragments([256]), 16)
wl.items["head_pair"][0], wl.items["head_pair"][1] = 1, 0
items, segs = ops.upload_worklist(wl, q.device)
o = torch.empty_like(q); lse = torch.empty(32, 256, device="cuda")
ops.attn_fwd(q, k, k, items, wl.n_items, segs, o, lse)
torch.cuda.synchronize()
print("NO ERROR")
'''
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert "NO ERROR" not in r.stdout and r.returncode != 0, r.stdout + r.stderr


def test_sm_reserve_leaves_results_bit_identical():
    """zp_attn_set_sm_reserve (SMs left free for ring-hop kernels) only caps the
    persistent grid: the output is bit-identical, and the previous value comes back."""
    seqlens = [3000, 700, 129]
    q, k, v = make_qkv(sum(seqlens), seed=11)
    o_full, lse_full = ops.varlen_attention(q, k, v, seqlens)
    prev = ops.set_sm_reserve(140)  # leaves only a few CTA pairs running
    try:
        o_cap, lse_cap = ops.varlen_attention(q, k, v, seqlens)
    finally:
        assert ops.set_sm_reserve(prev) == 140
    torch.cuda.synchronize()
    assert torch.equal(o_full, o_cap)
    assert torch.equal(lse_full, lse_cap)


def test_single_cta_kernel_gqa_group_of_two():
    """A GQA group of 2 (16 query / 8 KV heads) cannot pair head pairs of one
    KV head across a CTA pair, so it runs the single-CTA (cta_group::1) kernel."""
    seqlens = [1000, 130, 2049]
    t = sum(seqlens)
    q, k, v = make_qkv(t, hq=16, hkv=8, seed=21)
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    torch.cuda.synchronize()
    r = 0
    for n in seqlens:
        pos = torch.arange(n, device="cuda")
        ro, rl = ref_attention(q[r:r + n], k[r:r + n], v[r:r + n], pos, pos)
        assert (o[r:r + n].float() - ro).abs().max().item() <= MAX_ABS
        assert (lse[:, r:r + n] - rl).abs().max().item() <= 1e-2
        r += n


@pytest.mark.parametrize("hq,hkv,d", [(4, 4, 64), (4, 2, 64), (6, 2, 128), (8, 8, 96), (32, 8, 64)])
def test_other_head_shapes_through_the_adapter(hq, hkv, d):
    """BASELINE config 1's heads (4 x d64, MHA) and other shapes the kernel
    does not take natively run through ops.HeadAdapter (zero-padded head_dim,
    query heads duplicated for odd GQA groups), against fp32 with scale 1/sqrt(d)."""
    seqlens = [306, 66, 1, 241]
    t = sum(seqlens)
    g = torch.Generator().manual_seed(hq * 100 + d)
    q = torch.randn(t, hq, d, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(t, hkv, d, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(t, hkv, d, generator=g).to(torch.bfloat16).cuda()
    o, lse = ops.varlen_attention(q, k, v, seqlens)
    torch.cuda.synchronize()
    assert o.shape == q.shape and lse.shape == (hq, t)
    r = 0
    for n in seqlens:
        pos = torch.arange(n, device="cuda")
        ro, rl = ref_attention(q[r:r + n], k[r:r + n], v[r:r + n], pos, pos)
        assert (o[r:r + n].float() - ro).abs().max().item() <= MAX_ABS
        assert (lse[:, r:r + n] - rl).abs().max().item() <= 1e-2
        r += n
