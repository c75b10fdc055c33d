"""Config 5: a full Llama-3-8B transformer block on the Zeppelin layouts.

Where the reference models the block as "attention makespan + remap +
linear_per_token x tokens" (simulator.py:265-304), this executes it:

    x (linear layout, B_r rows)
      -> RMSNorm (zp_rmsnorm) -> QKV GEMM (cuBLAS)
      -> inverse remap of the qkv rows to the attention layout (fused peer-load kernel)
      -> RoPE at global in-sequence positions + q/k/v split (zp_rope_split)
      -> attention engine (zp_attn_fwd: local + ring rounds)
      -> forward remap of o to the linear layout (fused peer-load kernel)
      -> O GEMM + residual (cuBLAS addmm) -> RMSNorm -> gate/up GEMM
      -> SwiGLU (zp_swiglu) -> down GEMM + residual
    -> out (linear layout)

The linear modules run on the balanced linear layout, attention on the
attention layout (paper section 4.3; reference remapping.py).  GEMMs are plain
cuBLAS (torch.matmul / addmm in bf16 with fp32 accumulation) — the decision is
recorded in DESIGN.md; every other byte is moved by this repo's kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import engine, ops
from .plan import build_plan
from .program import build_rank_program
from .remap import solve_remap, cost_matrix
from .schedule import build_schedule

HIDDEN, HQ, HKV, HEAD_DIM, INTER = 4096, 32, 8, 128, 14336
ROPE_THETA, EPS = 500000.0, 1e-5


@dataclass
class BlockWeights:
    attn_norm: torch.Tensor  # [hidden]
    w_qkv: torch.Tensor      # [(hq + 2 hkv) * 128, hidden]
    w_o: torch.Tensor        # [hidden, hq * 128]
    mlp_norm: torch.Tensor   # [hidden]
    w_gu: torch.Tensor       # [2 * inter, hidden]  (gate rows, then up rows)
    w_down: torch.Tensor     # [hidden, inter]

    @classmethod
    def random(cls, device, seed: int = 0, hidden: int = HIDDEN, hq: int = HQ, hkv: int = HKV,
               inter: int = INTER) -> "BlockWeights":
        g = torch.Generator(device=device).manual_seed(seed)

        def lin(o, i):
            return (torch.randn(o, i, device=device, generator=g) / math.sqrt(i)).to(torch.bfloat16)

        def norm():
            return (1.0 + 0.1 * torch.randn(hidden, device=device, generator=g)).to(torch.bfloat16)

        return cls(norm(), lin((hq + 2 * hkv) * HEAD_DIM, hidden), lin(hidden, hq * HEAD_DIM), norm(),
                   lin(2 * inter, hidden), lin(hidden, inter))

    @property
    def inter(self) -> int:
        return self.w_down.shape[1]


def rope_tables(max_pos: int, device, theta: float = ROPE_THETA, d: int = HEAD_DIM):
    """cos/sin [max_pos, d/2] fp32, angle = pos * theta^(-2i/d) computed in fp64."""
    inv = theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return (torch.from_numpy(np.cos(ang).astype(np.float32)).to(device),
            torch.from_numpy(np.sin(ang).astype(np.float32)).to(device))


def attention_tokens(plan, rank: int) -> np.ndarray:
    """(sequence id, position) of every attention-layout row of a rank, [A_r, 2]."""
    parts = [np.stack([np.full(f.tokens, f.sequence_id, np.int64), np.arange(f.start, f.end)], 1)
             for f in plan.fragments[rank]]
    return np.concatenate(parts) if parts else np.zeros((0, 2), np.int64)


def linear_tokens(plan, layout, rank: int) -> np.ndarray:
    """(sequence id, position) of every linear-layout row of a rank, [B_r, 2]
    (the remap row rule applied to the attention-layout tokens)."""
    parts = [attention_tokens(plan, s)[o:o + n] for s, o, n in layout.source_of_linear_rows(rank)]
    return np.concatenate(parts) if parts else np.zeros((0, 2), np.int64)


def attention_positions(plan, rank: int) -> np.ndarray:
    """Global in-sequence position of every attention-layout row of a rank."""
    parts = [np.arange(f.start, f.end, dtype=np.int32) for f in plan.fragments[rank]]
    return np.concatenate(parts) if parts else np.zeros(0, np.int32)


class ZeppelinBlock:
    """One Llama-3-8B block for this rank (one process per GPU)."""

    def __init__(self, cluster, weights: BlockWeights, ctx: engine.RankContext | None = None,
                 max_pos: int = 262144, strategy: str = "zeppelin"):
        self.cluster = cluster
        self.strategy = strategy
        self.w = weights
        self.ctx = ctx or engine.RankContext.from_env()
        self.cos, self.sin = rope_tables(max_pos, self.ctx.device)
        self.hq = weights.w_o.shape[1] // HEAD_DIM
        self.hkv = (weights.w_qkv.shape[0] // HEAD_DIM - self.hq) // 2
        self.peer_qkv = self.peer_o = None
        if self.ctx.world > 1 and strategy == "zeppelin":
            cap = cluster.token_capacity
            self.peer_qkv = engine.PeerBuffer(self.ctx, cap, weights.w_qkv.shape[0])
            self.peer_o = engine.PeerBuffer(self.ctx, cap, self.hq * HEAD_DIM)

    def prepare(self, batch):
        r = self.ctx.rank
        if self.strategy == "zeppelin":
            self.plan = build_plan(batch, self.cluster)
            lay = solve_remap(self.plan.tokens_per_rank, cost_matrix(self.cluster))
        else:  # comparison strategies: no remap, linear modules on the attention layout
            from .baselines import plan_for
            from .remap import identity_layout
            self.plan = plan_for(self.strategy, batch, self.cluster)
            lay = identity_layout(self.plan.tokens_per_rank)
        self.schedule = build_schedule(self.plan)
        self.program = build_rank_program(self.plan, self.schedule, r, self.hq, lay)
        if not hasattr(self, "_stagers"):
            self._stagers = [engine.TableStager(self.ctx.device) for _ in range(3)]
        self.device_program = engine.DeviceProgram(self.program, self.ctx.device, self._stagers[0])
        self.layout = self.program.remap
        self.pos = self._stagers[1].upload(np.ascontiguousarray(attention_positions(self.plan, r)))
        # both remap tables of the step in one staged upload (no pinned allocation per call)
        self._pull = (engine.pull_table_pair(self.layout, r, self._stagers[2])
                      if self.peer_qkv is not None and self.layout.moved_rows() else (None, None))
        return self.plan

    @property
    def rows(self) -> tuple[int, int]:
        """(attention-layout rows A_r, linear-layout rows B_r)."""
        r = self.ctx.rank
        return self.layout.attn_rows[r], self.layout.linear_rows[r]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x [B_r, hidden] bf16 in the linear layout -> block output, same layout."""
        a, b = self.rows
        w, ctx = self.w, self.ctx
        if x.shape[0] != b:
            raise ValueError(f"rank {ctx.rank}: block input has {x.shape[0]} rows, linear layout has {b}")
        with ctx.span("compute", "linear", {"tokens": b, "op": "attn_norm+qkv"}):
            h = ops.rmsnorm(x, w.attn_norm, EPS)
            if self.peer_qkv is not None:
                qkv_buf = self.peer_qkv.buf
                torch.matmul(h, w.w_qkv.t(), out=qkv_buf[:b])
            else:
                qkv = torch.matmul(h, w.w_qkv.t())
        if self.peer_qkv is not None:
            engine.remap_pull(self.layout, self.peer_qkv, qkv_buf, ctx, inverse=True, tables=self._pull[1])
            qkv = qkv_buf[:a]
        with ctx.span("compute", "rope", {"tokens": a}):
            q, k, v = ops.rope_split(qkv, self.pos, self.cos, self.sin, self.hq, self.hkv)
        if self.peer_o is not None:
            o_buf = self.peer_o.buf
        else:
            o_buf = torch.empty(max(a, b, 1), self.hq * HEAD_DIM, dtype=torch.bfloat16, device=x.device)
        o = o_buf[:a].view(a, self.hq, HEAD_DIM)
        lse = torch.empty(self.hq, max(a, 1), dtype=torch.float32, device=x.device)
        engine.attention_forward(self.plan, self.schedule, q, k, v, ctx, self.program, self.device_program,
                                 out=(o, lse), kv_exchange="allgather" if self.strategy == "llama_cp" else "ring")
        if self.peer_o is not None:
            engine.remap_pull(self.layout, self.peer_o, o_buf, ctx, tables=self._pull[0])
            self._stagers[2].release()  # both readers of this step's remap tables are enqueued
        with ctx.span("compute", "linear", {"tokens": b, "op": "o+mlp"}):
            x2 = torch.addmm(x, o_buf[:b], w.w_o.t())
            h2 = ops.rmsnorm(x2, w.mlp_norm, EPS)
            gu = torch.matmul(h2, w.w_gu.t())
            act = ops.swiglu(gu)
            return torch.addmm(x2, act, w.w_down.t())

    def flops_per_step(self) -> tuple[int, int]:
        """(GEMM FLOPs, attention FLOPs) of this rank's step."""
        a, b = self.rows
        w = self.w
        gemm = 2 * b * (w.w_qkv.numel() + w.w_o.numel() + w.w_gu.numel() + w.w_down.numel())
        attn = 4 * HEAD_DIM * self.hq * self.program.pairs_per_head()
        return gemm, attn


def reference_block(x_seq: dict, w: BlockWeights, eps: float = EPS, theta: float = ROPE_THETA):
    """Plain PyTorch fp32 Llama block per sequence (the numerics reference for
    the GPU block; tests only).  x_seq: sid -> [len, hidden]."""
    out = {}
    f = {k: getattr(w, k).float() for k in ("attn_norm", "w_qkv", "w_o", "mlp_norm", "w_gu", "w_down")}
    hq = w.w_o.shape[1] // HEAD_DIM
    hkv = (w.w_qkv.shape[0] // HEAD_DIM - hq) // 2
    inter = w.inter

    def norm(t, g):
        return t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + eps) * g

    for sid, xs in x_seq.items():
        x = xs.float()
        n = x.shape[0]
        qkv = norm(x, f["attn_norm"]) @ f["w_qkv"].t()
        q = qkv[:, :hq * 128].view(n, hq, 128)
        k = qkv[:, hq * 128:(hq + hkv) * 128].view(n, hkv, 128)
        v = qkv[:, (hq + hkv) * 128:].view(n, hkv, 128)
        inv = theta ** (-torch.arange(0, 128, 2, dtype=torch.float64, device=x.device) / 128)
        ang = torch.arange(n, dtype=torch.float64, device=x.device)[:, None] * inv[None]
        cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]

        def rot(t):
            t1, t2 = t[..., :64], t[..., 64:]
            return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], -1)

        q, k = rot(q), rot(k)
        att = torch.nn.functional.scaled_dot_product_attention(
            q.transpose(0, 1), k.repeat_interleave(hq // hkv, 1).transpose(0, 1),
            v.repeat_interleave(hq // hkv, 1).transpose(0, 1), is_causal=True).transpose(0, 1)
        x2 = x + att.reshape(n, -1) @ f["w_o"].t()
        gu = norm(x2, f["mlp_norm"]) @ f["w_gu"].t()
        a = torch.nn.functional.silu(gu[:, :inter]) * gu[:, inter:]
        out[sid] = x2 + a @ f["w_down"].t()
    return out
