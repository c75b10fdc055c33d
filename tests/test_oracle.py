"""The CPU oracle itself: numerics pinned to torch's independent fp64 SDPA,
mask semantics pinned to the reference schedule's pair counts."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import remap as OR
from paper_2509_21841_b200 import plan as P, schedule as S, remap as M, workloads as W
from paper_2509_21841_b200.cluster import ClusterSpec
from paper_2509_21841_b200.batch import SequenceBatch


def rand_seqs(lengths, hq, hkv, d, seed):
    g = torch.Generator().manual_seed(seed)
    mk = lambda n, h: torch.randn(n, h, d, generator=g).to(torch.bfloat16).double().numpy()
    return ({s: mk(n, hq) for s, n in lengths}, {s: mk(n, hkv) for s, n in lengths},
            {s: mk(n, hkv) for s, n in lengths})


@pytest.mark.parametrize("n,hq,hkv,d", [(1, 4, 4, 64), (37, 4, 4, 64), (300, 8, 2, 32), (1500, 4, 1, 16)])
def test_causal_attention_matches_torch_sdpa_fp64(n, hq, hkv, d):
    q, k, v = (x[0] for x in rand_seqs([(0, n)], hq, hkv, d, n))
    pos = np.arange(n)
    o, lse, pairs = OA.causal_attention(q, k, v, pos, pos, d ** -0.5)
    assert pairs == S.causal_pairs(n)
    tq = torch.from_numpy(q).transpose(0, 1)
    tk = torch.from_numpy(k).repeat_interleave(hq // hkv, 1).transpose(0, 1)
    tv = torch.from_numpy(v).repeat_interleave(hq // hkv, 1).transpose(0, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True).transpose(0, 1).numpy()
    assert np.abs(o - ref).max() < 1e-12
    s = (tq @ tk.transpose(1, 2)) * d ** -0.5
    s = s.masked_fill(torch.ones(n, n, dtype=torch.bool).triu(1), float("-inf"))
    assert np.abs(lse - torch.logsumexp(s, -1).numpy()).max() < 1e-12


def _check_plan(plan, hq=4, hkv=4, d=64, seed=0):
    sched = S.build_schedule(plan)
    lengths = sorted(plan.sequence_lengths.items())
    sq, sk, sv = rand_seqs(lengths, hq, hkv, d, seed)
    res, round_pairs = OA.run_plan(plan, sched, sq, sk, sv, d ** -0.5)
    for (ri, i, r), cnt in round_pairs.items():
        assert cnt == sched.rings()[ri].rounds[i][r].compute_pairs
    # merged rings / locals == full per-sequence causal attention
    for rank, (o, lse) in enumerate(res):
        for sid, a, b, row0 in OA.layout_rows(plan, rank):
            n = plan.sequence_lengths[sid]
            pos = np.arange(n)
            fo, fl, _ = OA.causal_attention(sq[sid], sk[sid], sv[sid], pos, pos, d ** -0.5)
            assert np.abs(o[row0:row0 + b - a] - fo[a:b]).max() < 1e-12
            assert np.abs(lse[:, row0:row0 + b - a] - fl[:, a:b]).max() < 1e-12
    return sched


def test_c1_tiny_layer_two_simulated_ranks():
    """BASELINE config 1: 4 heads x d64, 8 long-tailed sequences, world_size 2."""
    plan = P.build_plan(W.c1_batch(), W.c1_cluster())
    sched = _check_plan(plan)
    assert len(sched.rings()) == 1 and sched.rings()[0].ring.members == (0, 1)


@pytest.mark.parametrize("seed", range(6))
def test_random_ring_plans(seed):
    rng = np.random.default_rng(seed)
    g = int(rng.choice([2, 3, 4]))
    lengths = [int(x) for x in rng.integers(1, 300, size=int(rng.integers(2, 7)))]
    lengths[0] = int(rng.integers(200, 600))
    total = sum(lengths)
    cluster = ClusterSpec(1, g, -(-total * 105 // (100 * g)), 1.0, 1.0)
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), cluster)
    _check_plan(plan, hq=2, hkv=1, d=16, seed=seed)


def test_remap_oracle_roundtrip_and_rule():
    for counts in ([497, 489], [10, 0, 7, 3], [33112, 33112, 33112, 32137, 31091, 34325, 34239, 31016]):
        lay = M.remap_layout(counts)
        x = [np.arange(n)[:, None] + 1000000 * r for r, n in enumerate(counts)]
        y = OR.forward(x, lay.matrix)
        assert [len(t) for t in y] == list(lay.linear_rows)
        back = OR.inverse(y, lay.matrix, counts)
        assert all(np.array_equal(a, b) for a, b in zip(x, back))
        for r in range(len(counts)):
            blocks = lay.source_of_linear_rows(r)
            want = np.concatenate([x[s][o:o + n] for s, o, n in blocks])
            assert np.array_equal(want, y[r])
