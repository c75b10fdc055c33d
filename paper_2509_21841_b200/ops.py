"""Device entry points over the C ABI, taking torch tensors.

torch is used only for device memory and streams; every byte of attention or
remap data is produced by the sm_100a kernels in ``csrc/``.  Nothing here has a
CPU path: inputs must be CUDA tensors and the library must load.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native
from .worklist import BwdWorkList, QueryFragment, WorkList, build_bwd_worklist, build_worklist

HEAD_DIM = 128

# Instrumentation: number of native kernel launches issued, and an optional
# hook that receives CUDA events bracketing each attention launch (bench.py
# uses it to time the dominant kernel on its own stream).
_launches = 0
_hook = None


def reset_launch_count() -> None:
    global _launches
    _launches = 0


def launch_count() -> int:
    return _launches


def _count_launch(n: int = 1) -> None:
    global _launches
    _launches += n


def set_launch_hook(fn) -> None:
    global _hook
    _hook = fn


_workspaces: dict = {}


def _workspace(device: torch.device, stream: int) -> torch.Tensor:
    """Scratch for the persistent scheduler's work counter (torch-owned), one
    per (device, stream): launches on one stream reuse theirs in stream order,
    launches on different streams never share one."""
    key = (device.index, stream)
    ws = _workspaces.get(key)
    if ws is None:
        ws = torch.empty(16, dtype=torch.uint8, device=device)  # zeroed by each launch on its stream
        _workspaces[key] = ws
    return ws


def _stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _require_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if not t.is_cuda:
            raise RuntimeError("zeppelin-b200 ops run on CUDA tensors only (no CPU fallback)")


def upload_worklist(wl: WorkList, device: torch.device) -> tuple[torch.Tensor, torch.Tensor]:
    """Copy the item / segment tables to the device (one H2D each)."""
    items = torch.from_numpy(wl.items.view(np.int32).reshape(-1)).pin_memory().to(device, non_blocking=True)
    segs = torch.from_numpy(wl.segs.view(np.int32).reshape(-1)).pin_memory().to(device, non_blocking=True)
    return items, segs


def set_sm_reserve(sms: int) -> int:
    """SMs the attention launches leave free (zp_attn_set_sm_reserve);
    returns the previous value."""
    return int(_native.lib().zp_attn_set_sm_reserve(int(sms)))


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, items: torch.Tensor, n_items: int,
             segs: torch.Tensor, o: torch.Tensor, lse: torch.Tensor,
             state_o: torch.Tensor | None = None, state_ml: torch.Tensor | None = None,
             softmax_scale: float | None = None, stream: torch.cuda.Stream | None = None) -> None:
    """Launch zp_attn_fwd over a device work list.

    q: [Tq, Hq, 128] bf16, k/v: [Tk, Hkv, 128] bf16 views whose row stride may
    exceed Hkv*128 (interleaved ring buffers), o: [Tq, Hq, 128] bf16,
    lse: [Hq, Tq] fp32.  Parity mode (zp_attn_fwd_parity) when v is fp16 and
    o fp32: P staged as fp16, unrounded fp32 output."""
    _require_cuda(q, k, v, o, lse)
    tq, hq, d = q.shape
    tk, hkv, dk = k.shape
    if d != HEAD_DIM or dk != HEAD_DIM or v.shape != k.shape:
        raise ValueError("head_dim must be 128 and k/v must have equal shapes")
    parity = v.dtype == torch.float16
    if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or v.dtype not in (torch.bfloat16, torch.float16):
        raise ValueError("q/k must be bf16, v bf16 (or fp16 for the parity mode)")
    if o.dtype != (torch.float32 if parity else torch.bfloat16):
        raise ValueError("o must be bf16 (fp32 in the parity mode, v fp16)")
    if q.stride() != (hq * d, d, 1) or o.stride() != (hq * d, d, 1):
        raise ValueError("q and o must be row-contiguous [T, H, 128]")
    if k.stride()[1:] != (d, 1) or v.stride() != k.stride():
        raise ValueError("k/v must have contiguous heads and equal strides")
    if lse.dtype != torch.float32 or lse.shape[0] != hq:
        raise ValueError("lse must be fp32 [Hq, >=Tq]")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    st_o = state_o.data_ptr() if state_o is not None else None
    st_ml = state_ml.data_ptr() if state_ml is not None else None
    st_rows = int(state_o.shape[0]) if state_o is not None else 0
    global _launches
    _launches += 1
    if _hook is not None:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    sp = _stream_ptr(stream)
    _native.call("zp_attn_fwd_parity" if parity else "zp_attn_fwd", q.data_ptr(), k.data_ptr(), v.data_ptr(),
                 tq, tk, k.stride(0), hq, hkv, d, o.data_ptr(), lse.data_ptr(), lse.stride(0), items.data_ptr(),
                 n_items, segs.data_ptr(), st_o, st_ml, st_rows, scale, _workspace(q.device, sp).data_ptr(), sp)
    if _hook is not None:
        ev1.record()
        _hook("zp_attn_fwd", ev0, ev1)


def upload_bwd_worklist(wl: BwdWorkList, device: torch.device) -> tuple[torch.Tensor, torch.Tensor]:
    items = torch.from_numpy(wl.items.view(np.int32).reshape(-1)).pin_memory().to(device, non_blocking=True)
    qsegs = torch.from_numpy(wl.qsegs.view(np.int32).reshape(-1)).pin_memory().to(device, non_blocking=True)
    return items, qsegs


def attn_bwd_prep(o: torch.Tensor, dout: torch.Tensor, delta: torch.Tensor,
                  stream: torch.cuda.Stream | None = None) -> None:
    """delta [Hq, >=T] fp32 <- rowsum(dO * O) per (head, row) (zp_attn_bwd_prep)."""
    _require_cuda(o, dout, delta)
    t, hq, d = o.shape
    if dout.shape != o.shape or o.dtype != torch.bfloat16 or dout.dtype != torch.bfloat16:
        raise ValueError("o and dout must be bf16 tensors of equal shape")
    if not (o.is_contiguous() and dout.is_contiguous()) or delta.dtype != torch.float32 or delta.shape[0] != hq:
        raise ValueError("o/dout must be contiguous, delta fp32 [Hq, >=T]")
    _count_launch()
    _native.call("zp_attn_bwd_prep", o.data_ptr(), dout.data_ptr(), t, hq, d, delta.data_ptr(),
                 delta.stride(0), _stream_ptr(stream))


def attn_bwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, dout: torch.Tensor, lse: torch.Tensor,
             delta: torch.Tensor, dq: torch.Tensor, dk: torch.Tensor, dv: torch.Tensor, items: torch.Tensor,
             n_items: int, qsegs: torch.Tensor, softmax_scale: float | None = None,
             stream: torch.cuda.Stream | None = None) -> None:
    """Launch zp_attn_bwd over a device backward work list.

    q/dout [Tq, Hq, 128] bf16; k/v [Tk, Hkv, 128] bf16 (row stride may exceed
    Hkv*128); lse/delta fp32 [Hq, >=Tq]; dq fp32 [Tq, Hq, 128] (accumulated),
    dk/dv fp32 [Tk, Hkv, 128] contiguous."""
    _require_cuda(q, k, v, dout, lse, delta, dq, dk, dv)
    tq, hq, d = q.shape
    tk, hkv, _ = k.shape
    if dout.shape != q.shape or not dout.is_contiguous() or q.stride() != (hq * d, d, 1):
        raise ValueError("q and dout must be row-contiguous [T, H, 128] of equal shape")
    if k.stride()[1:] != (d, 1) or v.stride() != k.stride() or v.shape != k.shape:
        raise ValueError("k/v must have contiguous heads and equal strides")
    for t_, shape in ((dq, q.shape), (dk, k.shape), (dv, k.shape)):
        if t_.dtype != torch.float32 or t_.shape != shape or not t_.is_contiguous():
            raise ValueError("dq/dk/dv must be contiguous fp32 with the q/k shapes")
    if lse.stride() != delta.stride() or lse.dtype != torch.float32 or delta.dtype != torch.float32:
        raise ValueError("lse and delta must be fp32 with equal strides")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    _count_launch()
    if _hook is not None:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    _native.call("zp_attn_bwd", q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), tq, tk, k.stride(0),
                 hq, hkv, d, lse.data_ptr(), delta.data_ptr(), lse.stride(0), dq.data_ptr(), dk.data_ptr(),
                 dv.data_ptr(), items.data_ptr(), n_items, qsegs.data_ptr(), scale, _stream_ptr(stream))
    if _hook is not None:
        ev1.record()
        _hook("zp_attn_bwd", ev0, ev1)


def varlen_attention_backward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor,
                              lse: torch.Tensor, dout: torch.Tensor, seqlens,
                              softmax_scale: float | None = None):
    """Backward of ``varlen_attention`` (LocalTask queue of one rank).
    Returns (dq, dk, dv) bf16 in the input shapes."""
    _require_cuda(q, k, v, o, lse, dout)
    t, hq, d = q.shape
    hkv = k.shape[1]
    wl = build_bwd_worklist(local_fragments(seqlens), hkv)
    delta = torch.empty_like(lse)
    attn_bwd_prep(o, dout, delta)
    dq = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    dk = torch.zeros(k.shape, dtype=torch.float32, device=q.device)
    dv = torch.zeros(k.shape, dtype=torch.float32, device=q.device)
    items, qsegs = upload_bwd_worklist(wl, q.device)
    attn_bwd(q, k, v, dout, lse, delta, dq, dk, dv, items, wl.n_items, qsegs, softmax_scale)
    return dq.to(torch.bfloat16), dk.to(torch.bfloat16), dv.to(torch.bfloat16)


def local_fragments(seqlens: list[int] | np.ndarray, row0: int = 0) -> list[QueryFragment]:
    """Whole-sequence causal fragments for sequences packed back to back."""
    frags = []
    r = row0
    for n in seqlens:
        n = int(n)
        frags.append(QueryFragment(row0=r, pos0=0, length=n, segs=[(r, 0, n)]))
        r += n
    return frags


class HeadAdapter:
    """Maps any attention head shape onto the kernel's (head_dim 128, even
    GQA group): head_dim d < 128 is zero-padded (q.k and the softmax are
    unchanged with the scale kept at 1/sqrt(d); the padded output columns are
    exact zeros and dropped), and an odd group (MHA: hq == hkv) is made even
    by running every query head twice against its KV head (outputs of the
    copies are identical; one is kept).  BASELINE config 1 (4 heads x d64,
    MHA) runs through this."""

    def __init__(self, hq: int, hkv: int, d: int):
        if d > HEAD_DIM or hq % hkv:
            raise ValueError(f"unsupported head shape: hq={hq} hkv={hkv} head_dim={d} (need d <= 128, hkv | hq)")
        self.hq, self.hkv, self.d = hq, hkv, d
        self.dup = 2 if (hq // hkv) % 2 else 1

    @property
    def identity(self) -> bool:
        return self.d == HEAD_DIM and self.dup == 1

    def inputs(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
        pad = HEAD_DIM - self.d
        if pad:
            q, k, v = (torch.nn.functional.pad(x, (0, pad)) for x in (q, k, v))
        if self.dup > 1:
            q = q.repeat_interleave(self.dup, dim=1)
        return q.contiguous(), k.contiguous(), v.contiguous()

    def outputs(self, o: torch.Tensor, lse: torch.Tensor):
        if self.dup > 1:
            o, lse = o[:, ::self.dup], lse[::self.dup]
        return o[..., :self.d].contiguous(), lse.contiguous()


def varlen_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seqlens,
                     softmax_scale: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Causal attention of packed variable-length sequences (all GPU-local):
    the LocalTask queue of one rank.  Returns (o bf16 [T,Hq,d], lse fp32 [Hq,T]);
    with an fp16 v the parity mode runs and o is fp32.  Any head_dim <= 128
    and any GQA group (HeadAdapter)."""
    _require_cuda(q, k, v)
    ad = HeadAdapter(q.shape[1], k.shape[1], q.shape[2])
    if not ad.identity:
        scale = 1.0 / math.sqrt(q.shape[2]) if softmax_scale is None else softmax_scale
        o, lse = varlen_attention(*ad.inputs(q, k, v), seqlens, softmax_scale=scale)
        return ad.outputs(o, lse)
    t, hq, _ = q.shape
    hkv = k.shape[1]
    wl = build_worklist(local_fragments(seqlens), hq // 2)
    o = torch.empty(q.shape, dtype=torch.float32 if v.dtype == torch.float16 else q.dtype, device=q.device)
    lse = torch.empty(hq, t, dtype=torch.float32, device=q.device)
    items, segs = upload_worklist(wl, q.device)
    attn_fwd(q, k, v, items, wl.n_items, segs, o, lse, softmax_scale=softmax_scale)
    return o, lse


def copy_rows(dst: torch.Tensor, src: torch.Tensor, ranges: torch.Tensor, n_ranges: int,
              max_rows: int, stream: torch.cuda.Stream | None = None) -> None:
    """dst[d0:d0+n] = src[s0:s0+n] for each (d0, s0, n) row of the int32
    device table ``ranges``; rows are the leading dimension of both tensors."""
    global _launches
    _require_cuda(dst, src, ranges)
    _launches += 1
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else dst[0].numel() * dst.element_size()
    _native.call("zp_copy_rows", dst.data_ptr(), dst.stride(0) * dst.element_size(), src.data_ptr(),
                 src.stride(0) * src.element_size(), row_bytes, ranges.data_ptr(), n_ranges,
                 max_rows, _stream_ptr(stream))


def add_f32_(dst: torch.Tensor, src: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """dst += src (contiguous fp32 of equal size), zp_add_f32."""
    _require_cuda(dst, src)
    if dst.dtype != torch.float32 or src.dtype != torch.float32 or dst.numel() != src.numel():
        raise ValueError("add_f32_: fp32 tensors of equal size")
    if not (dst.is_contiguous() and src.is_contiguous()):
        raise ValueError("add_f32_: contiguous tensors")
    _count_launch()
    _native.call("zp_add_f32", dst.data_ptr(), src.data_ptr(), dst.numel(), _stream_ptr(stream))


# ---------------------------------------------------------------- block kernels

def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-5, out: torch.Tensor | None = None) -> torch.Tensor:
    _require_cuda(x, w)
    y = out if out is not None else torch.empty_like(x)
    _count_launch()
    _native.call("zp_rmsnorm", x.data_ptr(), w.data_ptr(), y.data_ptr(), x.shape[0], x.shape[1], eps,
                 _stream_ptr())
    return y


def rope_split(qkv: torch.Tensor, pos: torch.Tensor, cos_t: torch.Tensor, sin_t: torch.Tensor,
               hq: int, hkv: int):
    """qkv [rows, (hq+2hkv)*128] -> q [rows,hq,128], k/v [rows,hkv,128] (q, k rotated)."""
    _require_cuda(qkv, pos, cos_t, sin_t)
    rows = qkv.shape[0]
    q = torch.empty(rows, hq, 128, dtype=qkv.dtype, device=qkv.device)
    k = torch.empty(rows, hkv, 128, dtype=qkv.dtype, device=qkv.device)
    v = torch.empty_like(k)
    _count_launch()
    _native.call("zp_rope_split", qkv.data_ptr(), pos.data_ptr(), cos_t.data_ptr(), sin_t.data_ptr(),
                 q.data_ptr(), k.data_ptr(), v.data_ptr(), rows, hq, hkv, 128, _stream_ptr())
    return q, k, v


def swiglu(gu: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    _require_cuda(gu)
    rows, two_inter = gu.shape
    y = out if out is not None else torch.empty(rows, two_inter // 2, dtype=gu.dtype, device=gu.device)
    _count_launch()
    _native.call("zp_swiglu", gu.data_ptr(), y.data_ptr(), rows, two_inter // 2, _stream_ptr())
    return y
