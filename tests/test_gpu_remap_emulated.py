"""The shipped fused remap kernels (zp_remap_pull / zp_remap_push and their
ready/done epoch handshakes) with every rank emulated on ONE B200: each rank
has its own stream and landing buffer, peers are reached through plain device
pointers instead of CUDA-IPC mappings, and the rows each rank ends up with
are compared with the CPU oracle (oracle/remap.py: the R3 row rule on the
reference's transfer matrix M, remapping.py:187-245; inverse = the exact
reverse, remapping.py:248-255).  Bit-exact: the payload is (rank, row) ids
plus random bf16 rows of the Llama-3 hidden size."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import remap as OR
from paper_2509_21841_b200 import plan as P, workloads as W
from paper_2509_21841_b200.emulate import emulate_remap_on_one_gpu
from paper_2509_21841_b200.remap import cost_matrix, remap_layout, solve_remap


def _ids(attn_rows):
    """16-byte rows: (rank, row, 0, 0) int32."""
    out = []
    for r, n in enumerate(attn_rows):
        t = torch.zeros(n, 4, dtype=torch.int32)
        t[:, 0] = r
        t[:, 1] = torch.arange(n, dtype=torch.int32)
        out.append(t.cuda())
    return out


def _layouts():
    cases = []
    for g in (2, 4, 8):
        batch = W.c4_batch(total=65536)
        cluster = W.cluster_for(batch, g)
        plan = P.build_plan(batch, cluster)
        res = solve_remap(plan.tokens_per_rank, cost_matrix(cluster))
        cases.append((f"plan_g{g}", remap_layout(plan.tokens_per_rank, res)))
    total = 16384
    for g in (2, 4, 8):
        cases.append((f"S1_fan_out_g{g}", remap_layout([total] + [0] * (g - 1))))
        cases.append((f"S2_alternating_g{g}", remap_layout([2 * total // g if i % 2 == 0 else 0 for i in range(g)])))
    cases.append(("ragged_g3", remap_layout([5000, 1, 77])))
    return cases


CASES = _layouts()


@pytest.mark.parametrize("method", ["pull", "push"])
@pytest.mark.parametrize("name,lay", CASES, ids=[c[0] for c in CASES])
def test_fused_remap_matches_oracle_permutation(name, lay, method):
    assert lay.moved_rows() > 0
    xs = _ids(lay.attn_rows)
    ys = emulate_remap_on_one_gpu(lay, xs, method)
    want = OR.source_map(list(lay.attn_rows), lay.matrix)
    for r in range(lay.world):
        assert ys[r].shape[0] == lay.linear_rows[r]
        assert np.array_equal(ys[r][:, :2].cpu().numpy(), want[r]), (name, method, r)
    back = emulate_remap_on_one_gpu(lay, ys, method, inverse=True)
    for r in range(lay.world):
        assert torch.equal(back[r], xs[r]), (name, method, r)


@pytest.mark.parametrize("method,total,g", [("pull", 65536, 4), ("push", 65536, 4), ("pull", 262144, 8)])
def test_fused_remap_hidden_4096_round_trip(method, total, g):
    """Config-4 row size (hidden 4096 bf16 = 8 KiB per token) on plan
    layouts, up to config 4's full 256K tokens over 8 ranks: forward equals
    the oracle's numpy move, inverse restores x."""
    batch = W.c4_batch(total=total)
    cluster = W.cluster_for(batch, g)
    plan = P.build_plan(batch, cluster)
    lay = remap_layout(plan.tokens_per_rank, solve_remap(plan.tokens_per_rank, cost_matrix(cluster)))
    gen = torch.Generator(device="cuda").manual_seed(5)
    xs = [torch.randn(n, 4096, device="cuda", generator=gen, dtype=torch.bfloat16) for n in lay.attn_rows]
    ys = emulate_remap_on_one_gpu(lay, xs, method)
    want = OR.forward([x.view(torch.int16).cpu().numpy() for x in xs], lay.matrix)
    for r in range(lay.world):
        assert np.array_equal(ys[r].view(torch.int16).cpu().numpy(), want[r])
    back = emulate_remap_on_one_gpu(lay, ys, method, inverse=True)
    for r in range(lay.world):
        assert torch.equal(back[r], xs[r])


def test_spin_timeout_traps_instead_of_hanging():
    """A rank whose peer never arrives: the ready handshake gives up after the
    configured bound with a message and a trap (the context dies, the GPU does
    not hang).  Child process: a trapped kernel poisons its CUDA context."""
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2509_21841_b200 import _native
from paper_2509_21841_b200.engine import PeerBuffer, RankContext, pull_tables, remap_pull
from paper_2509_21841_b200.remap import remap_layout
_native.lib().zp_set_spin_timeout_ms(2000)
lay = remap_layout([100, 0])
ctxs = [RankContext(r, 2, torch.device("cuda", 0)) for r in range(2)]
bufs = PeerBuffer.local_group(ctxs, 100, 4, torch.int32)
t = pull_tables(lay, 1, False, torch.device("cuda", 0))
remap_pull(lay, bufs[1], bufs[1].buf, ctxs[1], tables=t)   # rank 0 never calls
torch.cuda.synchronize()
print("NO ERROR")
'''
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert "NO ERROR" not in r.stdout and r.returncode != 0, r.stdout + r.stderr
    assert "handshake timed out" in r.stdout + r.stderr, r.stdout + r.stderr
