"""Chunked fp32 GPU reference for causal GQA attention (test infrastructure).

Plain PyTorch fp32 on the same bf16-rounded inputs the kernel reads: for each
block of query rows, S = q K^T * scale over the keys up to the block's last
row, causal mask (key position <= query position, reference
attention_engine.py:113-136), row softmax, P V — with TF32 disabled, so every
product and sum is IEEE fp32.  Query blocks keep the [block, keys] score
matrix a few GB even for 128K-token sequences; the 4 query heads of a GQA
group share one K/V head without expanding K/V.  Pinned to the fp64 CPU
oracle (oracle/attention.py) on spot rows by the parity tests.
"""

from __future__ import annotations

import torch


def causal_attention_fp32(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float | None = None,
                          block: int = 256) -> tuple[torch.Tensor, torch.Tensor]:
    """One whole sequence (positions 0..n-1).  q [n, Hq, d], k/v [n, Hkv, d]
    (any float dtype, on a CUDA device).  Returns (o fp32 [n, Hq, d],
    lse fp32 [Hq, n], natural log)."""
    n, hq, d = q.shape
    hkv = k.shape[1]
    g = hq // hkv
    scale = d ** -0.5 if scale is None else scale
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        kf = k.float().permute(1, 0, 2).contiguous()   # [hkv, n, d]
        vf = v.float().permute(1, 0, 2).contiguous()
        o = torch.empty(n, hq, d, dtype=torch.float32, device=q.device)
        lse = torch.empty(hq, n, dtype=torch.float32, device=q.device)
        for c0 in range(0, n, block):
            c1 = min(n, c0 + block)
            m = c1 - c0
            # [hkv, g*m, d]: row j*m + i = query row c0+i of head kvh*g + j
            qc = q[c0:c1].float().view(m, hkv, g, d).permute(1, 2, 0, 3).reshape(hkv, g * m, d)
            s = torch.bmm(qc, kf[:, :c1].transpose(1, 2)).mul_(scale).view(hkv, g, m, c1)
            diag = torch.ones(m, m, dtype=torch.bool, device=q.device).triu_(1)  # key > query
            s[..., c0:c1].masked_fill_(diag, float("-inf"))
            ls = torch.logsumexp(s, dim=-1)                                      # [hkv, g, m]
            p = torch.exp(s.sub_(ls[..., None]))
            oc = torch.bmm(p.view(hkv, g * m, c1), vf[:, :c1])                 # [hkv, g*m, d]
            o[c0:c1] = oc.view(hkv, g, m, d).permute(2, 0, 1, 3).reshape(m, hq, d)
            lse[:, c0:c1] = ls.reshape(hq, m)
            del s, p
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return o, lse


def causal_attention_backward_fp32(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, dout: torch.Tensor,
                                   scale: float | None = None, block: int = 256
                                   ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Gradients of ``causal_attention_fp32`` for one whole sequence, in
    plain fp32 (TF32 off), blockwise over query rows: the reference's own O
    and LSE, Delta = rowsum(dO * O), then per query block P = exp(S - LSE),
    dS = P * (dO V^T - Delta), dQ = scale * dS K, dK += scale * dS^T Q,
    dV += P^T dO.  Returns (dq [n, Hq, d], dk, dv [n, Hkv, d]) fp32."""
    n, hq, d = q.shape
    hkv = k.shape[1]
    g = hq // hkv
    scale = d ** -0.5 if scale is None else scale
    o, lse = causal_attention_fp32(q, k, v, scale, block)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        kf = k.float().permute(1, 0, 2).contiguous()   # [hkv, n, d]
        vf = v.float().permute(1, 0, 2).contiguous()
        delta = (dout.float() * o).sum(-1).transpose(0, 1).contiguous()  # [hq, n]
        dq = torch.empty(n, hq, d, dtype=torch.float32, device=q.device)
        dk = torch.zeros(hkv, n, d, dtype=torch.float32, device=q.device)
        dv = torch.zeros(hkv, n, d, dtype=torch.float32, device=q.device)
        for c0 in range(0, n, block):
            c1 = min(n, c0 + block)
            m = c1 - c0
            # [hkv, g*m, d]: row j*m + i = query row c0+i of head kvh*g + j
            grp = lambda t: t[c0:c1].float().view(m, hkv, g, d).permute(1, 2, 0, 3).reshape(hkv, g * m, d)  # noqa: E731
            qc, doc = grp(q), grp(dout)
            s = torch.bmm(qc, kf[:, :c1].transpose(1, 2)).mul_(scale).view(hkv, g, m, c1)
            diag = torch.ones(m, m, dtype=torch.bool, device=q.device).triu_(1)  # key > query
            s[..., c0:c1].masked_fill_(diag, float("-inf"))
            p = torch.exp(s.sub_(lse[:, c0:c1].reshape(hkv, g, m, 1))).view(hkv, g * m, c1)
            del s
            dp = torch.bmm(doc, vf[:, :c1].transpose(1, 2))                     # [hkv, g*m, c1]
            dp.sub_(delta[:, c0:c1].reshape(hkv, g * m, 1)).mul_(p)             # dS
            dq[c0:c1] = (torch.bmm(dp, kf[:, :c1]) * scale).view(hkv, g, m, d).permute(2, 0, 1, 3).reshape(m, hq, d)
            dk[:, :c1] += torch.bmm(dp.transpose(1, 2), qc) * scale
            dv[:, :c1] += torch.bmm(p.transpose(1, 2), doc)
            del p, dp
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return dq, dk.permute(1, 0, 2).contiguous(), dv.permute(1, 0, 2).contiguous()


class ErrorStats:
    """Accumulates the north-star error measures of an output against the
    fp32 reference: max |o - r|, mean-rel = sum |o - r| / sum |r|,
    signed bias = sum (o - r) / sum |r|, and max LSE error."""

    def __init__(self):
        self.max_abs = 0.0
        self.sum_abs_err = 0.0
        self.sum_err = 0.0
        self.sum_abs_ref = 0.0
        self.lse_max_abs = 0.0
        self.elements = 0

    def add(self, o: torch.Tensor, ref: torch.Tensor, lse: torch.Tensor | None = None,
            lse_ref: torch.Tensor | None = None) -> None:
        d = o.double() - ref.double()
        self.max_abs = max(self.max_abs, float(d.abs().max()))
        self.sum_abs_err += float(d.abs().sum())
        self.sum_err += float(d.sum())
        self.sum_abs_ref += float(ref.double().abs().sum())
        self.elements += ref.numel()
        if lse is not None:
            self.lse_max_abs = max(self.lse_max_abs, float((lse.double() - lse_ref.double()).abs().max()))

    @property
    def mean_rel(self) -> float:
        return self.sum_abs_err / max(self.sum_abs_ref, 1e-300)

    @property
    def bias(self) -> float:
        return self.sum_err / max(self.sum_abs_ref, 1e-300)

    def as_dict(self) -> dict:
        return {"max_abs": self.max_abs, "mean_rel": self.mean_rel, "signed_bias": self.bias,
                "lse_max_abs": self.lse_max_abs, "elements": self.elements}
