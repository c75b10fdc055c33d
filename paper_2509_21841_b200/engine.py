"""Device executor: runs a rank's program (``program.py``) on its B200.

One process per GPU.  Compute goes to the caller's current CUDA stream; the
ring KV exchange goes to a dedicated communication stream as copy-engine pulls
from the predecessor's CUDA-IPC-mapped buffer, ordered by epoch flags that the
stream front-end waits on (``RingTransport``, ``zp_ring_hop``: no SM, no
collective library), triple-buffered so round r's attention overlaps the
transfer of the next sets.  Rings run in ``schedule.rings()`` order on every
rank, so rings that share ranks are entered in the same order everywhere
(deadlock-free); a rank never waits on a ring it is not in.

Public entry points (drop-in execution of what the reference only costs):

* ``attention_forward(plan, schedule, q, k, v)`` — LocalTask + RingRound
  attention for this rank (reference simulator.py:124-188 charges it);
* ``remap_forward(layout, x)`` / ``remap_inverse(layout, y)`` — the
  attention<->linear token remap (simulator.py:282-302, remapping.py:187-255);
* ``attention_backward(plan, schedule, q, k, v, o, lse, dout)`` — its
  backward: LocalTask + RingRound gradients, dK/dV of a
  ring's KV sets travelling with them around the ring and returned to their
  owner with one extra hop (the reference charges g sends, README.md:119-124);
  the remap's backward is the transposed move (``remap_inverse`` /
  ``remap_forward`` of the gradient, remapping.py:248-255);
* ``ZeppelinLayer`` — plan + attention + remap for one batch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

import torch
import torch.distributed as dist

from . import ops
from .plan import build_plan
from .program import BwdProgram, RankProgram, build_bwd_program, build_rank_program
from .remap import RemapLayout, cost_matrix, solve_remap
from .schedule import build_schedule
from .worklist import BwdWorkList, WorkList


_CONTEXTS: dict = {}


class RankContext:
    """Rank identity, process group, streams and reusable device workspaces."""

    def __init__(self, rank: int = 0, world: int = 1, device: torch.device | None = None, group=None):
        if not torch.cuda.is_available():
            raise RuntimeError("zeppelin-b200 executes on CUDA devices only (no CPU fallback)")
        self.rank = rank
        self.world = world
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.comm_stream = torch.cuda.Stream(self.device) if world > 1 else None
        self._ws: dict[str, torch.Tensor] = {}
        self.tracer = None  # trace.Tracer: measured timeline in the reference trace schema
        # ring KV exchange (RingTransport): buffers + flags reachable by the peers,
        # and the epoch base of the next attention call (advanced identically on
        # every rank: the schedule is the same everywhere)
        self.ring: RingTransport | None = None
        self.ring_epoch = 16

    def span(self, stream_name: str, kind: str, payload: dict | None = None, stream=None):
        import contextlib
        if self.tracer is None:
            return contextlib.nullcontext()
        return self.tracer.span(stream_name, kind, payload, stream)

    @classmethod
    def from_env(cls) -> "RankContext":
        """The process's context for the default group on the current device
        (one per (rank, world, device), reused across calls: a context owns
        streams, workspaces and the IPC-registered ring buffers)."""
        if dist.is_available() and dist.is_initialized():
            key = (dist.get_rank(), dist.get_world_size(), torch.cuda.current_device())
        else:
            key = (0, 1, torch.cuda.current_device())
        ctx = _CONTEXTS.get(key)
        if ctx is None:
            ctx = cls(key[0], key[1], torch.device("cuda", key[2]))
            _CONTEXTS[key] = ctx
        return ctx

    def workspace(self, name: str, shape, dtype) -> torch.Tensor:
        numel = int(np.prod(shape))
        buf = self._ws.get(name)
        if buf is None or buf.numel() < numel or buf.dtype != dtype:
            buf = torch.empty(max(numel, 1), dtype=dtype, device=self.device)
            self._ws[name] = buf
        return buf[:numel].view(*shape)


@dataclass
class _DevWork:
    items: torch.Tensor
    segs: torch.Tensor
    n: int
    in_place: "_DevWork | None" = None  # ring round 0: the same items reading k / v in place


class TableStager:
    """Reusable pinned staging + device buffers for per-step work-list uploads.

    Allocating pinned memory every step (``tensor.pin_memory()``) and copying
    on the compute stream ties the host to the device's progress and breaks
    host-fed pipelines.  Here K slots rotate; each upload is a copy on a
    private stream that waits only for the kernels that read the slot K
    uploads ago; the compute stream waits for the copy.  The host blocks only
    if it runs K uploads ahead of the device.

    A slot counts as consumed when ``release()`` is called (the caller has
    enqueued every kernel that reads it) or, failing that, at the next
    upload — so a caller that uploads several tables for one step must pack
    them into one upload or release explicitly after the readers."""

    def __init__(self, device: torch.device, slots: int = 3):
        self.device = device
        self.slots = [None] * slots
        self.turn = 0
        self.prev = None
        self.stream = torch.cuda.Stream(device)

    def release(self) -> None:
        """Every reader of the latest upload is enqueued on the current stream."""
        if self.prev is not None and not self.prev["released"]:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self.prev["consumed"] = ev
            self.prev["released"] = True

    def upload(self, host: np.ndarray) -> torch.Tensor:
        cs = torch.cuda.current_stream(self.device)
        self.release()  # implicit: readers of the previous upload are enqueued by now
        n = host.size
        slot = self.slots[self.turn]
        self.turn = (self.turn + 1) % len(self.slots)
        if slot is None or slot["pin"].numel() < n:
            cap = max(n, 1 << 16)
            slot = {"pin": torch.empty(cap, dtype=torch.int32).pin_memory(),
                    "dev": torch.empty(cap, dtype=torch.int32, device=self.device),
                    "copied": None, "consumed": torch.cuda.Event(), "released": False}
            # the new block comes from the compute stream's pool: kernels still
            # in flight there may have used this memory — the copy waits for them
            slot["consumed"].record(cs)
            self.slots[self.turn - 1] = slot
        if slot["copied"] is not None:
            slot["copied"].synchronize()  # the previous copy out of this pinned slot is done
        slot["pin"][:n].numpy()[:] = host
        dev = slot["dev"][:n]
        with torch.cuda.stream(self.stream):
            if slot["consumed"] is not None:
                self.stream.wait_event(slot["consumed"])
            dev.copy_(slot["pin"][:n], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.stream)
        slot["copied"] = done
        slot["released"] = False
        cs.wait_event(done)
        self.prev = slot
        return dev


class DeviceProgram:
    """A RankProgram's int32 tables, uploaded with one pinned H2D copy."""

    def __init__(self, prog: RankProgram, device: torch.device, stager: TableStager | None = None):
        self.prog = prog
        chunks: list[np.ndarray] = []

        def add(arr: np.ndarray) -> tuple[int, int]:
            flat = np.ascontiguousarray(arr).view(np.int32).reshape(-1)
            off = sum(c.size for c in chunks)
            chunks.append(flat)
            return off, flat.size

        def add_work(wl: WorkList):
            return add(wl.items), add(wl.segs), wl.n_items

        local = add_work(prog.local)
        rings = []
        for rp in prog.rings:
            pack = add(rp.pack_ranges)
            rounds = [(add_work(rr.work), add_work(rr.work_in_place) if rr.work_in_place is not None else None)
                      for rr in rp.rounds]
            rings.append((pack, rounds))
        host = np.concatenate(chunks) if chunks else np.zeros(1, np.int32)
        if stager is not None:
            self.table = stager.upload(host)
        else:
            self.table = torch.from_numpy(host).pin_memory().to(device, non_blocking=True)

        def view(span):
            off, n = span
            return self.table[off:off + n]

        def dev_work(w, ip=None):
            a, b, n = w
            return _DevWork(view(a), view(b), n, dev_work(ip) if ip is not None else None)

        self.local = dev_work(local)
        self.rings = [(view(pack), [dev_work(w, ip) for w, ip in rounds]) for pack, rounds in rings]
        self.h2d_bytes = host.nbytes


class RingTransport:
    """One rank's ring KV buffers and epoch flags, plus the peers' addresses.

    ``n_buf`` buffers of ``rows`` KV rows (K and V interleaved per row, 4 KiB
    per token at Llama-3 shapes) in one allocation, and an int32 flag block
    ``[0, world)`` "KV set full from predecessor p", ``[world, 2*world)`` "KV
    set consumed by successor s", ``[2*world, 3*world)`` "dK/dV partial sum
    ready from predecessor p", ``[3*world, 4*world)`` "partial sum consumed by
    successor s" (the last two for the backward's gradient buffers, attached
    on the first backward call).  Peers reach everything over NVLink through
    CUDA IPC (``create`` / ``attach_grad``, collective), or — ranks emulated in
    one process on one GPU — through plain device pointers (``local_group``).
    A hop is ``zp_ring_hop``: stream-ordered flag waits / writes and one
    copy-engine pull, no SM (RingHop describes the protocol)."""

    N_BUF = 3

    def __init__(self, ctx: RankContext, rows: int, row_bytes: int):
        self.ctx = ctx
        self.rows, self.row_bytes = rows, row_bytes
        self.storage = torch.empty(self.N_BUF * max(rows, 1) * row_bytes, dtype=torch.uint8, device=ctx.device)
        self.flags = torch.zeros(4 * ctx.world, dtype=torch.int32, device=ctx.device)
        self.buf_base: list[int] = []   # per rank: address of its storage (this process's mapping)
        self.flag_base: list[int] = []  # per rank: address of its flag block
        self.gstorage: torch.Tensor | None = None  # N_GRAD fp32 dK/dV partial-sum buffers
        self.grad_base: list[int] = []
        self.grad_rows = 0
        self.grad_elems = 0  # hkv * d

    def fits(self, rows: int, row_bytes: int) -> bool:
        return rows <= self.rows and row_bytes == self.row_bytes

    @classmethod
    def create(cls, ctx: RankContext, rows: int, row_bytes: int) -> "RingTransport":
        """Collective over ctx.group: allocate and exchange IPC handles."""
        t = cls(ctx, rows, row_bytes)
        torch.cuda.synchronize(ctx.device)
        mine = (_ipc_export(t.storage), _ipc_export(t.flags))
        everyone = [None] * ctx.world
        dist.all_gather_object(everyone, mine, group=ctx.group)
        for r, ((bh, bo), (fh, fo)) in enumerate(everyone):
            if r == ctx.rank:
                t.buf_base.append(t.storage.data_ptr())
                t.flag_base.append(t.flags.data_ptr())
            else:
                t.buf_base.append(_ipc_open(bh, bo))
                t.flag_base.append(_ipc_open(fh, fo))
        dist.barrier(group=ctx.group)
        return t

    @classmethod
    def local_group(cls, ctxs: list[RankContext], rows: int, row_bytes: int) -> list["RingTransport"]:
        """Emulated ranks on one device: peers' buffers are local pointers."""
        ts = [cls(c, rows, row_bytes) for c in ctxs]
        for t in ts:
            t.buf_base = [x.storage.data_ptr() for x in ts]
            t.flag_base = [x.flags.data_ptr() for x in ts]
        return ts

    def buffer(self, j: int, hkv: int, d: int) -> torch.Tensor:
        n = self.rows * self.row_bytes
        return self.storage[j * n:(j + 1) * n].view(torch.bfloat16).view(self.rows, 2, hkv, d)

    N_GRAD = 3

    def _grad_alloc(self, rows: int, elems: int) -> None:
        self.grad_rows, self.grad_elems = rows, elems
        self.gstorage = torch.empty(self.N_GRAD * 2 * max(rows, 1) * elems, dtype=torch.float32,
                                    device=self.ctx.device)

    def grad_fits(self, rows: int, elems: int) -> bool:
        return self.gstorage is not None and rows <= self.grad_rows and elems == self.grad_elems

    def attach_grad(self, rows: int, elems: int) -> None:
        """Collective: allocate this rank's dK/dV partial-sum buffers and
        exchange their IPC handles."""
        self._grad_alloc(rows, elems)
        ctx = self.ctx
        torch.cuda.synchronize(ctx.device)
        everyone = [None] * ctx.world
        dist.all_gather_object(everyone, _ipc_export(self.gstorage), group=ctx.group)
        self.grad_base = [self.gstorage.data_ptr() if r == ctx.rank else _ipc_open(h, o)
                          for r, (h, o) in enumerate(everyone)]
        dist.barrier(group=ctx.group)

    @staticmethod
    def attach_grad_local(ts: list["RingTransport"], rows: int, elems: int) -> None:
        for t in ts:
            t._grad_alloc(rows, elems)
        for t in ts:
            t.grad_base = [x.gstorage.data_ptr() for x in ts]

    def grad_buffer(self, j: int, hkv: int, d: int) -> torch.Tensor:
        """[2 (dK, dV), grad_rows, hkv, d] fp32 view of partial-sum buffer j."""
        n = 2 * self.grad_rows * self.grad_elems
        return self.gstorage[j * n:(j + 1) * n].view(2, self.grad_rows, hkv, d)

    def grad_addr(self, rank: int, j: int, half: int) -> int:
        """Address of rank's partial-sum buffer j, dK (half 0) or dV (half 1)."""
        return self.grad_base[rank] + 4 * self.grad_elems * self.grad_rows * (2 * j + half)

    def gfull_flag(self, owner: int, sender: int) -> int:
        return self.flag_base[owner] + 4 * (2 * self.ctx.world + sender)

    def gcons_flag(self, owner: int, reader: int) -> int:
        return self.flag_base[owner] + 4 * (3 * self.ctx.world + reader)

    def buf_addr(self, rank: int, j: int) -> int:
        return self.buf_base[rank] + j * self.rows * self.row_bytes

    def full_flag(self, owner: int, sender: int) -> int:
        """Address of owner's "full from sender" flag."""
        return self.flag_base[owner] + 4 * sender

    def consumed_flag(self, owner: int, reader: int) -> int:
        """Address of owner's "consumed by reader" flag."""
        return self.flag_base[owner] + 4 * (self.ctx.world + reader)


def ring_rows_needed(schedule) -> int:
    """KV buffer rows every rank allocates: the largest set any position of
    any ring holds (identical on every rank: taken from the global schedule,
    so a growth re-exchange is entered collectively)."""
    return max((rs.ring.kv_tokens(p) for rs in schedule.rings() for p in range(rs.ring.group_size)), default=0)


def _ensure_ring_transport(ctx: RankContext, schedule, hkv: int, d: int) -> RingTransport:
    rows = ring_rows_needed(schedule)
    row_bytes = 2 * hkv * d * 2
    if ctx.ring is None or not ctx.ring.fits(rows, row_bytes):
        grow = rows if ctx.ring is None else max(rows, int(1.25 * ctx.ring.rows))
        ctx.ring = RingTransport.create(ctx, grow, row_bytes)
    return ctx.ring


def _pack_and_announce(ctx: RankContext, rp, epoch0: int, dev_pack, k, v, bufs) -> None:
    """Own KV set -> transport buffer 0, announced to the successor (epoch
    offset 0); this ring's hops start after the pack (event edge): they
    refill buffers the previous ring's rounds read, and their flag writes
    must land after the pack's (a flag only grows)."""
    from . import _native
    T, xs = ctx.ring, ctx.comm_stream
    n_pack = rp.pack_ranges.shape[0]
    max_pack = int(rp.pack_ranges[:, 2].max()) if n_pack else 0
    cs = torch.cuda.current_stream()
    ops.copy_rows(bufs[0][:, 0], k, dev_pack, n_pack, max_pack)
    ops.copy_rows(bufs[0][:, 1], v, dev_pack, n_pack, max_pack)
    _native.call("zp_stream_write_flag", T.full_flag(rp.next_rank, ctx.rank), epoch0, int(cs.cuda_stream))
    packed = torch.cuda.Event()
    packed.record(cs)
    xs.wait_event(packed)


def _kv_hop(ctx: RankContext, rp, epoch0: int, h, done: dict) -> torch.cuda.Event:
    """Hop h (program.RingHop) on the comm stream: the predecessor's set
    -> own buffer h.dst_buf.  Returns the event the round that reads it waits
    for."""
    from . import _native
    T, xs = ctx.ring, ctx.comm_stream
    me, pred, succ = ctx.rank, rp.prev_rank, rp.next_rank
    if h.free is not None:
        xs.wait_event(done[h.free])  # the dst buffer's last local reader
    if ctx.tracer is not None:
        # traced step: wait for the flags first, so the span times the copy alone
        _native.call("zp_stream_wait_flag", T.full_flag(me, pred), epoch0 + h.full, int(xs.cuda_stream))
        if h.free is not None:
            _native.call("zp_stream_wait_flag", T.consumed_flag(me, succ), epoch0 + h.free, int(xs.cuda_stream))
    with ctx.span("intra-comm", "kv.send", {"ring": rp.ring_index, "round": h.round_index, "tokens": h.rows,
                                             "bytes": h.rows * T.row_bytes, "src": pred}, xs):
        _native.call("zp_ring_hop", T.buf_addr(me, h.dst_buf), T.buf_addr(pred, h.src_buf),
                     h.rows * T.row_bytes, T.full_flag(me, pred), epoch0 + h.full,
                     T.consumed_flag(me, succ) if h.free is not None else None,
                     epoch0 + (h.free or 0), T.consumed_flag(pred, me), epoch0 + h.consumed,
                     T.full_flag(succ, me) if h.next_full is not None else None,
                     epoch0 + (h.next_full or 0), int(xs.cuda_stream))
    ev = torch.cuda.Event()
    ev.record(xs)
    return ev


def _leave_ring(ctx: RankContext, rp, epoch0: int) -> None:
    """Leave the ring only after the successor pulled its last set from us
    (the next ring refills buffer 0); later work on the compute stream waits."""
    from . import _native
    xs = ctx.comm_stream
    if rp.group_size >= 2:
        _native.call("zp_stream_wait_flag", ctx.ring.consumed_flag(ctx.rank, rp.next_rank),
                     epoch0 + rp.group_size - 2, int(xs.cuda_stream))
    torch.cuda.current_stream().wait_stream(xs)


def _ring_steps(ctx: RankContext, rp, epoch0: int, dev_pack, dev_rounds, q, k, v, o, lse, scale,
                pack_after: torch.cuda.Event | None = None):
    """One ring at this position, as a generator: yields after the pack and
    after each round is enqueued (the single-GPU emulation interleaves the
    members' generators step by step, so every flag wait is enqueued after
    the write it waits for).  Compute on the current stream, the pack and the
    hops on the context's comm stream (copy engines; no SM is taken from the
    rounds).

    Per round r: attention of this position's query rows against the KV set
    held from position (i - r) mod g (reference attention_engine.py:229-244),
    resuming the running softmax state; hop r pulls the next set from the
    predecessor (attention_engine.py:247-251) while round r runs.  Round 0
    (the position's own set) reads k / v in place, so it starts while the set
    is being packed for the successor."""
    from . import _native
    T = ctx.ring
    hkv, d = k.shape[1], k.shape[2]
    hq = q.shape[1]
    g, me, succ = rp.group_size, ctx.rank, rp.next_rank
    xs = ctx.comm_stream
    parity = v.dtype == torch.float16
    bufs = [T.buffer(j, hkv, d) for j in range(rp.n_buffers)]
    st_o = ctx.workspace("ring_state_o", (max(rp.state_rows, 1), hq, d), torch.float32)
    st_ml = ctx.workspace("ring_state_ml", (2, hq, max(rp.state_rows, 1)), torch.float32)
    # own set -> buffer 0 on the comm stream, announced to the successor
    # (epoch offset 0); the hops follow on the same stream, so their flag
    # writes land after the pack's (a flag only grows)
    cs = torch.cuda.current_stream()
    if pack_after is None:
        pack_after = torch.cuda.Event()
        pack_after.record(cs)  # k / v final; the previous ring's rounds no longer read buffer 0
    xs.wait_event(pack_after)
    n_pack = rp.pack_ranges.shape[0]
    max_pack = int(rp.pack_ranges[:, 2].max()) if n_pack else 0
    ops.copy_rows(bufs[0][:, 0], k, dev_pack, n_pack, max_pack, stream=xs)
    ops.copy_rows(bufs[0][:, 1], v, dev_pack, n_pack, max_pack, stream=xs)
    _native.call("zp_stream_write_flag", T.full_flag(succ, me), epoch0, int(xs.cuda_stream))
    yield
    hops = rp.hops()
    ready: dict[int, torch.cuda.Event] = {}
    done: dict[int, torch.cuda.Event] = {}
    for r in range(g):
        cs = torch.cuda.current_stream()
        if r < g - 1:
            ready[r + 1] = _kv_hop(ctx, rp, epoch0, hops[r], done)
        if r > 0:
            cs.wait_event(ready[r])
        work = dev_rounds[r]
        with ctx.span("compute", "intra_node.attn",
                      {"ring": rp.ring_index, "round": r, "pairs": rp.rounds[r].work.pairs_per_head}):
            if r == 0 and work.in_place is not None:
                w = work.in_place
                if w.n:
                    ops.attn_fwd(q, k, v, w.items, w.n, w.segs, o, lse, st_o, st_ml, softmax_scale=scale)
            elif work.n:
                buf = bufs[r % rp.n_buffers]
                n_kv = rp.rounds[r].kv_rows
                vv = buf[:n_kv, 1].view(torch.float16) if parity else buf[:n_kv, 1]
                ops.attn_fwd(q, buf[:n_kv, 0], vv, work.items, work.n, work.segs, o, lse, st_o, st_ml,
                             softmax_scale=scale)
        ev = torch.cuda.Event()
        ev.record(cs)
        done[r] = ev
        yield
    _leave_ring(ctx, rp, epoch0)


def _run_ring_allgather(ctx: RankContext, rp, dev_pack, dev_rounds, q, k, v, o, lse, scale):
    """LLaMA-CP style execution of a ring (reference baselines.py:114-117,
    simulator.py:227-262): every member all-gathers the ring's KV sets first
    (one NCCL all-gather, not overlapped), then runs all rounds back to back."""
    hkv, d = k.shape[1], k.shape[2]
    hq = q.shape[1]
    g = rp.group_size
    rows = max(rp.held_rows)
    gathered = ctx.workspace("ring_allgather", (g, rows, 2, hkv, d), torch.bfloat16)
    mine = ctx.workspace("ring_allgather_mine", (rows, 2, hkv, d), torch.bfloat16)
    st_o = ctx.workspace("ring_state_o", (max(rp.state_rows, 1), hq, d), torch.float32)
    st_ml = ctx.workspace("ring_state_ml", (2, hq, max(rp.state_rows, 1)), torch.float32)
    n_pack = rp.pack_ranges.shape[0]
    max_pack = int(rp.pack_ranges[:, 2].max()) if n_pack else 0
    ops.copy_rows(mine[:, 0], k, dev_pack, n_pack, max_pack)
    ops.copy_rows(mine[:, 1], v, dev_pack, n_pack, max_pack)
    if g != ctx.world or tuple(rp.members) != tuple(range(ctx.world)):
        raise ValueError("all-gather KV exchange needs a ring over every rank (LLaMA-CP layout)")
    with ctx.span("intra-comm", "kv.allgather", {"tokens": int(rp.held_rows[rp.position])}):
        dist.all_gather_into_tensor(gathered, mine, group=ctx.group)
    for r in range(g):
        work = dev_rounds[r]
        buf = gathered[rp.rounds[r].src_position]
        n_kv = rp.rounds[r].kv_rows
        if work.n:
            ops.attn_fwd(q, buf[:n_kv, 0], buf[:n_kv, 1], work.items, work.n, work.segs, o, lse,
                         st_o, st_ml, softmax_scale=scale)


def attention_steps(plan, schedule, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, ctx: RankContext,
                    prog: RankProgram, devp: "DeviceProgram", o: torch.Tensor, lse: torch.Tensor, scale: float,
                    kv_exchange: str = "ring"):
    """Generator form of ``attention_forward``: yields ``(ring_index, step)``
    after each ring step (pack = step 0, round r = step r+1).  Rings run in
    ``schedule.rings()`` order on every rank (reference attention_engine.py:
    266-271), each position pulling the next KV set while it computes; local
    tasks fill the waits the reference's executor model predicts before each
    ring and the rest run after the last ring (program.local_fill_plan)."""
    epoch = ctx.ring_epoch
    ctx.ring_epoch += 16 * len(schedule.rings())  # the same on every rank
    done = 0
    # the first ring's pack needs only the inputs: it does not wait for the
    # local work queued before the ring
    inputs_ready = torch.cuda.Event()
    inputs_ready.record(torch.cuda.current_stream())

    def local_items(upto: int):
        # LocalTask items [done, upto) of the longest-first list (zp_attn_fwd)
        nonlocal done
        if upto > done:
            w = devp.local
            with ctx.span("compute", "local.attn", {"items": upto - done}):
                ops.attn_fwd(q, k, v, w.items[8 * done:8 * upto], upto - done, w.segs, o, lse, softmax_scale=scale)
            done = upto

    for j, (rp, (pack, rounds)) in enumerate(zip(prog.rings, devp.rings)):
        # local work that fills this rank's predicted wait for the ring's
        # slowest member (program.local_fill_plan), then the ring
        local_items(prog.local_cuts[j] if j < len(prog.local_cuts) else done)
        if kv_exchange == "allgather":
            _run_ring_allgather(ctx, rp, pack, rounds, q, k, v, o, lse, scale)
            continue
        for step, _ in enumerate(_ring_steps(ctx, rp, epoch + 16 * rp.ring_index, pack, rounds, q, k, v, o,
                                             lse, scale, pack_after=inputs_ready if j == 0 else None)):
            yield rp.ring_index, step
    local_items(devp.local.n)  # what is left runs after the last ring (simulator.py:181-187)


def attention_forward(plan, schedule, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                      ctx: RankContext | None = None, program: RankProgram | None = None,
                      device_program: DeviceProgram | None = None, softmax_scale: float | None = None,
                      out: tuple[torch.Tensor, torch.Tensor] | None = None, kv_exchange: str = "ring"):
    """This rank's attention (LocalTasks + every RingRound it takes part in).

    q [A_r, Hq, 128], k/v [A_r, Hkv, 128] bf16 in the rank's attention layout
    (plan.fragments[rank] rows in order).  Returns (o [A_r, Hq, 128] bf16,
    lse [Hq, A_r] fp32).  With an fp16 v the parity mode runs (fp16 P/V,
    fp32 o; ``zp_attn_fwd_parity``).  Collective when the plan has rings:
    every rank of the context calls it with the same plan."""
    ctx = ctx or RankContext.from_env()
    ad = ops.HeadAdapter(q.shape[1], k.shape[1], q.shape[2])
    if not ad.identity:
        # other head shapes (e.g. BASELINE config 1: 4 heads x d64, MHA) run on
        # the padded / head-duplicated layout the kernel supports
        scale = 1.0 / math.sqrt(q.shape[2]) if softmax_scale is None else softmax_scale
        o2, lse2 = attention_forward(plan, schedule, *ad.inputs(q, k, v), ctx=ctx, softmax_scale=scale,
                                     kv_exchange=kv_exchange)
        o, lse = ad.outputs(o2, lse2)
        if out is not None:
            out[0].copy_(o)
            out[1][:, :lse.shape[1]].copy_(lse)
            return out
        return o, lse
    hq = q.shape[1]
    prog = program or build_rank_program(plan, schedule, ctx.rank, hq)
    if q.shape[0] != prog.rows or k.shape[0] != prog.rows:
        raise ValueError(f"rank {ctx.rank}: expected {prog.rows} attention-layout rows, got {q.shape[0]}")
    devp = device_program or DeviceProgram(prog, q.device)
    scale = 1.0 / math.sqrt(q.shape[2]) if softmax_scale is None else softmax_scale
    if out is None:
        o = torch.empty(q.shape, dtype=torch.float32 if v.dtype == torch.float16 else q.dtype, device=q.device)
        lse = torch.empty(hq, max(prog.rows, 1), dtype=torch.float32, device=q.device)
    else:
        o, lse = out
    if ctx.world > 1 and schedule.rings() and kv_exchange == "ring":
        _ensure_ring_transport(ctx, schedule, k.shape[1], k.shape[2])
    for _ in attention_steps(plan, schedule, q, k, v, ctx, prog, devp, o, lse, scale, kv_exchange):
        pass
    return o, lse


# ------------------------------------------------------------------ backward

class BwdDeviceProgram:
    """A BwdProgram's int32 tables, uploaded with one pinned H2D copy."""

    def __init__(self, bp: BwdProgram, device: torch.device):
        self.bp = bp
        chunks: list[np.ndarray] = []

        def add(arr: np.ndarray) -> tuple[int, int]:
            flat = np.ascontiguousarray(arr).view(np.int32).reshape(-1)
            off = sum(c.size for c in chunks)
            chunks.append(flat)
            return off, flat.size

        def add_work(wl: BwdWorkList):
            return add(wl.items), add(wl.qsegs), wl.n_items

        local = add_work(bp.local)
        rings = [([add_work(wl) for wl in lists], add(up)) for lists, up in zip(bp.rounds, bp.unpack_ranges)]
        host = np.concatenate(chunks) if chunks else np.zeros(1, np.int32)
        self.table = torch.from_numpy(host).pin_memory().to(device, non_blocking=True)

        def view(span):
            off, n = span
            return self.table[off:off + n]

        self.local = _DevWork(view(local[0]), view(local[1]), local[2])
        self.rings = [([_DevWork(view(a), view(b), n) for a, b, n in rounds], view(up)) for rounds, up in rings]


def _ring_bwd_steps(ctx: RankContext, rp, epoch0: int, dev_pack, dev_rounds, dev_unpack, q, k, v, dout, lse,
                    delta, dq, dk, dv, scale):
    """Ring backward at this position, as a generator (steps as in
    ``_ring_steps``).  The KV sets travel exactly as in the forward.  Round r
    computes dQ (accumulated in place) and this position's share Z_r of the
    dK/dV of the set it holds, into partial-sum buffer r % 3.  On the comm
    stream, once round r is done, the running total A_r of that set is pulled
    from the predecessor (its buffer of round r-1, a copy-engine read over
    NVLink), added (T_r = Z_r + A_r, ``zp_add_f32``) and announced to the
    successor, which pulls it for round r+1; after the last round the
    predecessor's total of this position's own set is pulled and unpacked into
    dk / dv — the reference charges g sends per ring (README.md:119-124), the
    backward uses all of them.  The compute stream never waits for gradients,
    except before refilling a partial-sum buffer the successor has not pulled
    yet (three buffers)."""
    from . import _native
    T = ctx.ring
    hkv, d = k.shape[1], k.shape[2]
    g, me, pred, succ = rp.group_size, ctx.rank, rp.prev_rank, rp.next_rank
    xs = ctx.comm_stream
    xsp = int(xs.cuda_stream)
    bufs = [T.buffer(j, hkv, d) for j in range(rp.n_buffers)]
    gz = [T.grad_buffer(j, hkv, d) for j in range(T.N_GRAD)]
    ga = [ctx.workspace(f"ring_ga{j}", (2, T.grad_rows, hkv, d), torch.float32) for j in (0, 1)]
    half = T.grad_elems * 4  # bytes per row of one half (dK or dV)
    _pack_and_announce(ctx, rp, epoch0, dev_pack, k, v, bufs)
    yield
    hops = rp.hops()
    ready: dict[int, torch.cuda.Event] = {}
    done: dict[int, torch.cuda.Event] = {}

    def pull_total(r_src: int, rows: int, into: torch.Tensor) -> None:
        # the predecessor's running total of its round r_src (buffer r_src % 3)
        _native.call("zp_stream_wait_flag", T.gfull_flag(me, pred), epoch0 + r_src, xsp)
        for hf in (0, 1):
            _native.call("zp_memcpy_async", into[hf].data_ptr(), T.grad_addr(pred, r_src % T.N_GRAD, hf),
                         rows * half, xsp)
        _native.call("zp_stream_write_flag", T.gcons_flag(pred, me), epoch0 + r_src, xsp)

    for r in range(g):
        cs = torch.cuda.current_stream()
        if r < g - 1:
            ready[r + 1] = _kv_hop(ctx, rp, epoch0, hops[r], done)
        if r > 0:
            cs.wait_event(ready[r])
        n_kv = rp.rounds[r].kv_rows
        z = gz[r % T.N_GRAD]
        if r >= T.N_GRAD:  # the successor pulled what this buffer held (T_{r-3})
            _native.call("zp_stream_wait_flag", T.gcons_flag(me, succ), epoch0 + r - T.N_GRAD,
                         int(cs.cuda_stream))
        for hf in (0, 1):
            _native.call("zp_memset_async", z[hf].data_ptr(), 0, n_kv * half, int(cs.cuda_stream))
        work = dev_rounds[r]
        buf = bufs[r % rp.n_buffers]
        with ctx.span("compute", "intra_node.attn_bwd",
                      {"ring": rp.ring_index, "round": r, "pairs": rp.rounds[r].work.pairs_per_head}):
            if work.n:
                ops.attn_bwd(q, buf[:n_kv, 0], buf[:n_kv, 1], dout, lse, delta, dq, z[0][:n_kv], z[1][:n_kv],
                             work.items, work.n, work.segs, softmax_scale=scale)
        ev = torch.cuda.Event()
        ev.record(cs)
        done[r] = ev
        # running total of the held set: + what the previous holders accumulated
        xs.wait_event(ev)
        with ctx.span("intra-comm", "dkv.send", {"ring": rp.ring_index, "round": r, "tokens": n_kv}, xs):
            if r > 0:
                a = ga[r % 2]
                pull_total(r - 1, n_kv, a)
                ops.add_f32_(z[0][:n_kv], a[0][:n_kv], stream=xs)
                ops.add_f32_(z[1][:n_kv], a[1][:n_kv], stream=xs)
            _native.call("zp_stream_write_flag", T.gfull_flag(succ, me), epoch0 + r, xsp)
        yield
    # this position's own set: its total arrives from the predecessor's last round
    own = rp.held_rows[rp.position]
    a = ga[g % 2]
    pull_total(g - 1, own, a)
    n_up = dev_unpack.numel() // 3
    if n_up:
        max_up = int(rp.pack_ranges[:, 2].max())
        ops.copy_rows(dk, a[0], dev_unpack, n_up, max_up, stream=xs)
        ops.copy_rows(dv, a[1], dev_unpack, n_up, max_up, stream=xs)
    yield  # (step g+1: every member has pulled its own total)
    # the successor pulled our last total too, before the buffers are reused
    _native.call("zp_stream_wait_flag", T.gcons_flag(me, succ), epoch0 + g - 1, xsp)
    _leave_ring(ctx, rp, epoch0)


def _ensure_ring_grad(ctx: RankContext, schedule, hkv: int, d: int) -> None:
    rows = ring_rows_needed(schedule)
    T = ctx.ring
    if not T.grad_fits(rows, hkv * d):
        T.attach_grad(max(rows, int(1.25 * T.grad_rows)) if T.gstorage is not None else rows, hkv * d)


def attention_backward_steps(plan, schedule, q, k, v, dout, lse, delta, dq, dk, dv, ctx: RankContext,
                             prog: RankProgram, bdev: "BwdDeviceProgram", devp: "DeviceProgram", scale: float):
    """Generator form of ``attention_backward`` (fp32 dq / dk / dv given):
    LocalTask gradients, then every ring in ``schedule.rings()`` order;
    yields ``(ring_index, step)`` with steps 0 (pack) .. g (rounds) and g+1
    (own total pulled)."""
    epoch = ctx.ring_epoch
    ctx.ring_epoch += 16 * len(schedule.rings())  # the same on every rank
    if bdev.local.n:
        with ctx.span("compute", "local.attn_bwd", {"pairs": bdev.bp.local.pairs_per_head}):
            ops.attn_bwd(q, k, v, dout, lse, delta, dq, dk, dv, bdev.local.items, bdev.local.n, bdev.local.segs,
                         softmax_scale=scale)
    for i, rp in enumerate(prog.rings):
        rounds, unpack = bdev.rings[i]
        for step, _ in enumerate(_ring_bwd_steps(ctx, rp, epoch + 16 * rp.ring_index, devp.rings[i][0], rounds,
                                                 unpack, q, k, v, dout, lse, delta, dq, dk, dv, scale)):
            yield rp.ring_index, step


def attention_backward(plan, schedule, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor,
                       lse: torch.Tensor, dout: torch.Tensor, ctx: RankContext | None = None,
                       program: RankProgram | None = None, bwd_program: BwdDeviceProgram | None = None,
                       softmax_scale: float | None = None):
    """Gradients of this rank's attention (the backward of ``attention_forward``
    with the same plan).  o / lse are the forward outputs (final LSE).
    Returns (dq, dk, dv) bf16 in the rank's attention layout.  Collective when
    the plan has rings (every rank calls it with the same plan)."""
    ctx = ctx or RankContext.from_env()
    hq, hkv = q.shape[1], k.shape[1]
    prog = program or build_rank_program(plan, schedule, ctx.rank, hq)
    if q.shape[0] != prog.rows or dout.shape != q.shape:
        raise ValueError(f"rank {ctx.rank}: expected {prog.rows} attention-layout rows")
    bdev = bwd_program or BwdDeviceProgram(build_bwd_program(prog, hkv), q.device)
    scale = 1.0 / math.sqrt(q.shape[2]) if softmax_scale is None else softmax_scale
    delta = torch.empty_like(lse)
    ops.attn_bwd_prep(o, dout, delta)
    dq = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    dk = torch.zeros(k.shape, dtype=torch.float32, device=q.device)
    dv = torch.zeros(k.shape, dtype=torch.float32, device=q.device)
    devp = DeviceProgram(prog, q.device)
    if ctx.world > 1 and schedule.rings():
        _ensure_ring_transport(ctx, schedule, hkv, k.shape[2])
        _ensure_ring_grad(ctx, schedule, hkv, k.shape[2])
    for _ in attention_backward_steps(plan, schedule, q, k, v, dout, lse, delta, dq, dk, dv, ctx, prog, bdev,
                                      devp, scale):
        pass
    return dq.to(torch.bfloat16), dk.to(torch.bfloat16), dv.to(torch.bfloat16)


# ------------------------------------------------------------------ remap

def _all_to_all(ctx: RankContext, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
    if ctx.world == 1:
        return
    dist.all_to_all_single(out, inp, output_split_sizes=[int(x) for x in out_splits],
                           input_split_sizes=[int(x) for x in in_splits], group=ctx.group)


def _copy_prefix(dst: torch.Tensor, src: torch.Tensor, n: int, ctx: RankContext) -> None:
    if n <= 0 or dst.data_ptr() == src.data_ptr():
        return
    host = torch.empty((1, 3), dtype=torch.int32, pin_memory=True)  # caching host allocator
    host[0, 0], host[0, 1], host[0, 2] = 0, 0, n
    ops.copy_rows(dst, src, host.to(dst.device, non_blocking=True), 1, n)


def _remap_move(ctx: RankContext, src: torch.Tensor, dst: torch.Tensor, slices, moved: int) -> None:
    kept, (s_lo, s_hi), (r_lo, r_hi), send, recv = slices
    _copy_prefix(dst, src, kept, ctx)
    # every rank enters (or skips) the collective together: the decision uses
    # the layout's global row count, never this rank's own send / recv
    if moved > 0:
        _all_to_all(ctx, dst[r_lo:r_hi], src[s_lo:s_hi], recv, send)


def remap_forward(layout: RemapLayout, x: torch.Tensor, ctx: RankContext | None = None,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """Attention layout [A_r, hidden] -> linear layout [B_r, hidden].

    Kept rows stay in place (no copy when ``out`` shares ``x``'s storage); the
    tail [B_r, A_r) leaves and received blocks land at [A_r, B_r) in sender
    order — both contiguous, so NCCL's all-to-allv moves them directly."""
    ctx = ctx or RankContext.from_env()
    a, b = layout.attn_rows[ctx.rank], layout.linear_rows[ctx.rank]
    if x.shape[0] != a:
        raise ValueError(f"rank {ctx.rank}: remap input has {x.shape[0]} rows, layout says {a}")
    y = out if out is not None else torch.empty((b,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    _remap_move(ctx, x, y, layout.forward_slices(ctx.rank), layout.moved_rows())
    return y


def remap_inverse(layout: RemapLayout, y: torch.Tensor, ctx: RankContext | None = None,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """Linear layout [B_r, hidden] -> attention layout [A_r, hidden] (exact inverse)."""
    ctx = ctx or RankContext.from_env()
    a, b = layout.attn_rows[ctx.rank], layout.linear_rows[ctx.rank]
    if y.shape[0] != b:
        raise ValueError(f"rank {ctx.rank}: remap input has {y.shape[0]} rows, layout says {b}")
    x = out if out is not None else torch.empty((a,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    _remap_move(ctx, y, x, layout.inverse_slices(ctx.rank), layout.moved_rows())
    return x


# ------------------------------------------------------------------ fused remap (peer stores)

_opened: dict[bytes, int] = {}


def _ipc_export(t: torch.Tensor) -> tuple[bytes, int]:
    """CUDA-IPC handle of the allocation holding ``t`` plus t's byte offset in it."""
    import ctypes
    from . import _native
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _native.check(_native.lib().zp_ipc_get_handle(t.data_ptr(), h, ctypes.byref(off)), "zp_ipc_get_handle")
    return h.raw, int(off.value)


def _ipc_open(handle: bytes, offset: int) -> int:
    base = _opened.get(handle)
    if base is None:
        import ctypes
        out = ctypes.c_void_p()
        from . import _native
        buf = ctypes.create_string_buffer(handle, 64)
        _native.check(_native.lib().zp_ipc_open_handle(buf, ctypes.byref(out)), "zp_ipc_open_handle")
        base = int(out.value)
        _opened[handle] = base
    return base + offset


class PeerBuffer:
    """A landing buffer every rank can store into over NVLink (CUDA IPC), with
    its int32[2*world] ready/done flag block.  Collective constructor."""

    def __init__(self, ctx: RankContext, rows: int, row_elems: int, dtype=torch.bfloat16):
        self.ctx = ctx
        self.buf = torch.empty(max(rows, 1), row_elems, dtype=dtype, device=ctx.device)
        self.flags = torch.zeros(2 * ctx.world, dtype=torch.int32, device=ctx.device)
        torch.cuda.synchronize(ctx.device)
        mine = (_ipc_export(self.buf), _ipc_export(self.flags))
        everyone = [None] * ctx.world
        dist.all_gather_object(everyone, mine, group=ctx.group)
        ptrs, fptrs = [], []
        for r, ((bh, bo), (fh, fo)) in enumerate(everyone):
            if r == ctx.rank:
                ptrs.append(self.buf.data_ptr())
                fptrs.append(self.flags.data_ptr())
            else:
                ptrs.append(_ipc_open(bh, bo))
                fptrs.append(_ipc_open(fh, fo))
        self.peer_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=ctx.device)
        self.flag_ptrs = torch.tensor(fptrs, dtype=torch.int64, device=ctx.device)
        self.epoch = 0
        self.host_ptrs = None
        dist.barrier(group=ctx.group)

    @property
    def row_bytes(self) -> int:
        return self.buf.shape[1] * self.buf.element_size()

    @classmethod
    def local_group(cls, ctxs: list[RankContext], rows: int, row_elems: int, dtype=torch.bfloat16):
        """Emulated ranks on one device: every peer pointer is a local one
        (same kernels and handshakes as the IPC-mapped buffers)."""
        out = []
        for c in ctxs:
            pb = cls.__new__(cls)
            pb.ctx = c
            pb.buf = torch.empty(max(rows, 1), row_elems, dtype=dtype, device=c.device)
            pb.flags = torch.zeros(2 * c.world, dtype=torch.int32, device=c.device)
            pb.epoch = 0
            pb.host_ptrs = None
            out.append(pb)
        ptrs = [pb.buf.data_ptr() for pb in out]
        fptrs = [pb.flags.data_ptr() for pb in out]
        for pb in out:
            pb.peer_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=pb.buf.device)
            pb.flag_ptrs = torch.tensor(fptrs, dtype=torch.int64, device=pb.buf.device)
        return out


@dataclass
class _PushTables:
    table: torch.Tensor  # int32 [4, world]: src_row0, dst_row0, count, expect/readers
    max_count: int
    host: np.ndarray | None = None  # same table on the host (copy-engine path)


def push_tables(layout: RemapLayout, rank: int, inverse: bool, device) -> _PushTables:
    """Per-destination rows for zp_remap_push (forward: attention -> linear)."""
    w = layout.world
    m = layout.matrix
    if not inverse:
        count = [int(m[rank, d]) for d in range(w)]
        src0 = layout.send_offsets(rank)
        dst0 = [layout.recv_offsets(d)[rank] for d in range(w)]
        expect = [int(m[s, rank] > 0) for s in range(w)]
    else:
        count = [int(m[d, rank]) for d in range(w)]
        src0 = layout.recv_offsets(rank)
        dst0 = [layout.send_offsets(d)[rank] for d in range(w)]
        expect = [int(m[rank, s] > 0) for s in range(w)]
    host = torch.tensor([src0, dst0, count, expect], dtype=torch.int32)
    return _PushTables(host.pin_memory().to(device, non_blocking=True), max(count) if count else 0,
                       np.ascontiguousarray(host.numpy()))


def remap_push(layout: RemapLayout, x: torch.Tensor, peer: PeerBuffer, ctx: RankContext,
               inverse: bool = False, tables: _PushTables | None = None,
               copy_engine: bool = False, phases: int = 7) -> torch.Tensor:
    """Fused remap: this rank's outgoing rows are stored straight into the
    receivers' ``peer`` buffers (one kernel, NVLink peer stores, ready/done
    epoch flags) — the all-to-allv without a collective library.  Kept rows
    are copied only if ``x`` is not already ``peer.buf``'s prefix.  Returns the
    local landing view (linear layout for forward, attention layout for
    inverse)."""
    from . import _native
    r = ctx.rank
    a, b = layout.attn_rows[r], layout.linear_rows[r]
    rows_in, rows_out = (b, a) if inverse else (a, b)
    if x.shape[0] != rows_in:
        raise ValueError(f"rank {r}: remap input has {x.shape[0]} rows, layout says {rows_in}")
    out = peer.buf[:rows_out]
    if phases & 1:
        _copy_prefix(out, x, min(a, b), ctx)
    if layout.moved_rows() == 0:
        return out
    tb = tables or push_tables(layout, r, inverse, x.device)
    if phases & 1:
        peer.epoch += 1
    t = tb.table
    if copy_engine:
        if peer.host_ptrs is None:
            peer.host_ptrs = np.ascontiguousarray(peer.peer_ptrs.cpu().numpy())
        h = tb.host
        ops._count_launch(2)
        _native.call("zp_remap_push_ce", x.data_ptr(), peer.row_bytes, peer.host_ptrs.ctypes.data,
                     h[0].ctypes.data, h[1].ctypes.data, h[2].ctypes.data, peer.flag_ptrs.data_ptr(),
                     t[2].data_ptr(), t[3].data_ptr(), ctx.world, r, peer.epoch,
                     int(torch.cuda.current_stream().cuda_stream))
        return out
    ops._count_launch(bin(phases).count("1"))
    _native.call("zp_remap_push_phased", x.data_ptr(), peer.row_bytes, peer.peer_ptrs.data_ptr(),
                 t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), peer.flag_ptrs.data_ptr(),
                 t[3].data_ptr(), ctx.world, r, peer.epoch, tb.max_count, phases,
                 int(torch.cuda.current_stream().cuda_stream))
    return out


def _pull_host(layout: RemapLayout, rank: int, inverse: bool) -> np.ndarray:
    w = layout.world
    m = layout.matrix
    if not inverse:
        count = [int(m[s, rank]) for s in range(w)]
        src0 = [layout.send_offsets(s)[rank] for s in range(w)]
        dst0 = layout.recv_offsets(rank)
        readers = [int(m[rank, d] > 0) for d in range(w)]
    else:
        count = [int(m[rank, d]) for d in range(w)]
        src0 = [layout.recv_offsets(d)[rank] for d in range(w)]
        dst0 = layout.send_offsets(rank)
        readers = [int(m[s, rank] > 0) for s in range(w)]
    return np.asarray([src0, dst0, count, readers], dtype=np.int32)


def pull_table_pair(layout: RemapLayout, rank: int, stager: TableStager) -> tuple[_PushTables, _PushTables]:
    """Forward and inverse pull tables of one step in ONE staged upload (so
    the stager's slot is consumed only after both remaps were enqueued)."""
    fw, inv = _pull_host(layout, rank, False), _pull_host(layout, rank, True)
    w = layout.world
    dev = stager.upload(np.concatenate([fw.reshape(-1), inv.reshape(-1)])).view(2, 4, w)
    return (_PushTables(dev[0], int(fw[2].max()) if w else 0, np.ascontiguousarray(fw)),
            _PushTables(dev[1], int(inv[2].max()) if w else 0, np.ascontiguousarray(inv)))


def pull_tables(layout: RemapLayout, rank: int, inverse: bool, device,
                stager: TableStager | None = None) -> _PushTables:
    """Per-source rows for zp_remap_pull (forward: attention -> linear)."""
    w = layout.world
    m = layout.matrix
    if not inverse:
        count = [int(m[s, rank]) for s in range(w)]
        src0 = [layout.send_offsets(s)[rank] for s in range(w)]
        dst0 = layout.recv_offsets(rank)
        readers = [int(m[rank, d] > 0) for d in range(w)]
    else:
        count = [int(m[rank, d]) for d in range(w)]
        src0 = [layout.recv_offsets(d)[rank] for d in range(w)]
        dst0 = layout.send_offsets(rank)
        readers = [int(m[s, rank] > 0) for s in range(w)]
    host = torch.tensor([src0, dst0, count, readers], dtype=torch.int32)
    if stager is not None:
        dev = stager.upload(host.numpy().reshape(-1)).view(4, w)
    else:
        dev = host.pin_memory().to(device, non_blocking=True)
    return _PushTables(dev, max(count) if count else 0, np.ascontiguousarray(host.numpy()))


def remap_pull(layout: RemapLayout, src: PeerBuffer, out: torch.Tensor, ctx: RankContext,
               inverse: bool = False, tables: _PushTables | None = None,
               copy_engine: bool = False, phases: int = 7) -> torch.Tensor:
    """Fused remap, pull form: this rank reads its incoming rows straight from
    the senders' IPC-shared buffers (``src``: attention layout for forward,
    linear layout for inverse) over NVLink into ``out``.  ``phases`` (bit 1
    ready, 2 move, 4 done) splits the call for ranks emulated on one GPU."""
    from . import _native
    r = ctx.rank
    a, b = layout.attn_rows[r], layout.linear_rows[r]
    rows_in, rows_out = (b, a) if inverse else (a, b)
    if out.shape[0] < rows_out:
        raise ValueError(f"rank {r}: remap output needs {rows_out} rows")
    if phases & 1:
        _copy_prefix(out, src.buf[:rows_in], min(a, b), ctx)
    if layout.moved_rows() == 0:
        return out[:rows_out]
    tb = tables or pull_tables(layout, r, inverse, out.device)
    if phases & 1:
        src.epoch += 1
    t = tb.table
    stream = int(torch.cuda.current_stream().cuda_stream)
    if copy_engine:
        import ctypes
        if src.host_ptrs is None:
            src.host_ptrs = np.ascontiguousarray(src.peer_ptrs.cpu().numpy())
        h = tb.host
        ops._count_launch(2)
        _native.call("zp_remap_pull_ce", out.data_ptr(), src.row_bytes, src.host_ptrs.ctypes.data,
                     h[0].ctypes.data, h[1].ctypes.data, h[2].ctypes.data, src.flag_ptrs.data_ptr(),
                     t[2].data_ptr(), t[3].data_ptr(), ctx.world, r, src.epoch, stream)
        return out[:rows_out]
    ops._count_launch(bin(phases).count("1"))
    with ctx.span("intra-comm", "remap.inverse" if inverse else "remap.forward", {"tokens": int(tb.host[2].sum())}):
        _native.call("zp_remap_pull_phased", out.data_ptr(), src.row_bytes, src.peer_ptrs.data_ptr(),
                     t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), src.flag_ptrs.data_ptr(),
                     t[3].data_ptr(), ctx.world, r, src.epoch, tb.max_count, phases, stream)
    return out[:rows_out]


# ------------------------------------------------------------------ layer

class ZeppelinLayer:
    """Plan a batch and run attention + remap for this rank.

    ``prepare(batch)`` runs the host planner (bit-identical to the reference)
    and uploads this rank's work lists; ``forward(q, k, v)`` executes the
    attention engine and the remap to the balanced linear layout;
    ``backward_layout(y)`` restores the attention layout."""

    def __init__(self, cluster, ctx: RankContext | None = None, n_heads: int = 32, n_kv_heads: int = 8,
                 head_dim: int = 128, remap_method: str = "pull"):
        self.cluster = cluster
        self.ctx = ctx or RankContext.from_env()
        self.n_heads, self.n_kv_heads, self.head_dim = n_heads, n_kv_heads, head_dim
        self.plan = self.schedule = self.program = self.device_program = None
        if remap_method not in ("pull", "push", "nccl"):
            raise ValueError("remap_method must be 'pull', 'push' or 'nccl'")
        self.remap_method = remap_method
        self.peer: PeerBuffer | None = None

    def prepare(self, batch):
        self.plan = build_plan(batch, self.cluster)
        self.schedule = build_schedule(self.plan)
        # the reference's minimax transfer matrix for this cluster (remapping.py:187-245)
        remap = solve_remap(self.plan.tokens_per_rank, cost_matrix(self.cluster))
        self.program = build_rank_program(self.plan, self.schedule, self.ctx.rank, self.n_heads, remap)
        if not hasattr(self, "_stager"):
            self._stager = TableStager(self.ctx.device)
            self._remap_stager = TableStager(self.ctx.device)
        self.device_program = DeviceProgram(self.program, self.ctx.device, self._stager)
        self._pull = None
        if self.ctx.world > 1 and self.remap_method == "pull":
            self._pull = pull_table_pair(self.program.remap, self.ctx.rank, self._remap_stager)
        return self.plan

    @property
    def layout(self) -> RemapLayout:
        return self.program.remap

    def attention(self, q, k, v):
        return attention_forward(self.plan, self.schedule, q, k, v, self.ctx, self.program, self.device_program)

    # ------------------------------------------------------------ host-fed steps
    def step_host(self, q_h: torch.Tensor, k_h: torch.Tensor, v_h: torch.Tensor, o_h: torch.Tensor) -> None:
        """One layer step fed from pinned HOST buffers, pipelined: the H2D of
        this step's q/k/v runs on a copy stream while the previous step
        computes, and the D2H of the attention output (after the remap round
        trip) runs on a third stream while the next step computes.  Two device
        slots (inputs + activation buffer) alternate.  Asynchronous: call
        ``torch.cuda.synchronize()`` (or ``drain()``) before reading ``o_h``."""
        ctx = self.ctx
        dev = ctx.device
        rows, hq, d = q_h.shape
        if not hasattr(self, "_slots"):
            self._slots = []
            for _ in range(2):
                uses_peer = ctx.world > 1 and self.remap_method != "nccl"
                self._slots.append({"act": True if uses_peer else None, "free": torch.cuda.Event(),
                                    "used": False})
            self._h2d = torch.cuda.Stream(dev)
            self._d2h = torch.cuda.Stream(dev)
            self._turn = 0
        slot = self._slots[self._turn]
        self._turn ^= 1
        key = (rows, hq, k_h.shape[1], d)
        cs = torch.cuda.current_stream(dev)
        fresh = None
        if slot.get("key") != key:
            slot["q"] = torch.empty(rows, hq, d, dtype=torch.bfloat16, device=dev)
            slot["k"] = torch.empty(rows, k_h.shape[1], d, dtype=torch.bfloat16, device=dev)
            slot["v"] = torch.empty_like(slot["k"])
            if slot["act"] is None:
                slot["own_act"] = torch.empty(max(rows, max(self.layout.linear_rows), 1), hq * d,
                                              dtype=torch.bfloat16, device=dev)
            slot["key"] = key
            # fresh blocks come from the compute stream's pool; the copy stream
            # must not write them before earlier kernels there are done
            fresh = torch.cuda.Event()
            fresh.record(cs)
        ready = torch.cuda.Event()
        with torch.cuda.stream(self._h2d):
            if fresh is not None:
                self._h2d.wait_event(fresh)
            if slot["used"]:
                self._h2d.wait_event(slot["free"])  # step i-2 no longer reads this slot's inputs
            slot["q"].copy_(q_h, non_blocking=True)
            slot["k"].copy_(k_h, non_blocking=True)
            slot["v"].copy_(v_h, non_blocking=True)
            ready.record(self._h2d)
        cs.wait_event(ready)
        if slot["used"]:
            cs.wait_event(slot["d2h_done"])  # previous D2H of this slot's output finished
        q, k, v = slot["q"], slot["k"], slot["v"]
        if slot["act"] is not None:
            peer = slot["peer_obj"] if "peer_obj" in slot else None
            if peer is None:
                peer = self._peer_for(slot)
            act = peer.buf
            o = act[:rows].view(rows, hq, d)
            lse = torch.empty(hq, max(rows, 1), dtype=torch.float32, device=dev)
            attention_forward(self.plan, self.schedule, q, k, v, ctx, self.program, self.device_program,
                              out=(o, lse))
            if self.remap_method == "pull":
                fw, inv = self._pull or (None, None)
                remap_pull(self.layout, peer, act, ctx, tables=fw)
                remap_pull(self.layout, peer, act, ctx, inverse=True, tables=inv)
                self._remap_stager.release()  # both readers of this step's tables are enqueued
            else:
                remap_push(self.layout, act[:rows], peer, ctx)
                remap_push(self.layout, act[:self.layout.linear_rows[ctx.rank]], peer, ctx, inverse=True)
            res = act[:rows]
        else:
            act = slot["own_act"]
            o = act[:rows].view(rows, hq, d)
            lse = torch.empty(hq, max(rows, 1), dtype=torch.float32, device=dev)
            attention_forward(self.plan, self.schedule, q, k, v, ctx, self.program, self.device_program,
                              out=(o, lse))
            y = remap_forward(self.layout, act[:rows], ctx, out=act[:self.layout.linear_rows[ctx.rank]])
            res = remap_inverse(self.layout, y, ctx, out=act[:rows])
        slot["free"].record(cs)
        done = torch.cuda.Event()
        with torch.cuda.stream(self._d2h):
            self._d2h.wait_event(slot["free"])
            o_h.view(rows, -1).copy_(res, non_blocking=True)
            done.record(self._d2h)
        slot["d2h_done"] = done
        slot["used"] = True

    def _peer_for(self, slot) -> "PeerBuffer":
        peer = PeerBuffer(self.ctx, self.cluster.token_capacity, self.n_heads * self.head_dim)
        slot["peer_obj"] = peer
        slot["act"] = peer.buf
        return peer

    def activation_buffer(self) -> torch.Tensor:
        """[token_capacity, Hq*128] bf16 buffer shared over CUDA IPC (world > 1):
        attention output lands in its prefix [0, A_r) and the remap turns it
        into the linear layout [0, B_r) in place."""
        if self.peer is None and self.ctx.world > 1 and self.remap_method != "nccl":
            self.peer = PeerBuffer(self.ctx, self.cluster.token_capacity, self.n_heads * self.head_dim)
        return self.peer.buf if self.peer is not None else None

    def forward(self, q, k, v):
        """Attention in the attention layout, then remap to the balanced linear
        layout.  Returns (o, lse, y) with y [B_r, Hq*128]."""
        buf = self.activation_buffer()
        rows = q.shape[0]
        if buf is None:
            o, lse = self.attention(q, k, v)
            return o, lse, remap_forward(self.layout, o.view(rows, -1), self.ctx)
        o = buf[:rows].view(rows, self.n_heads, self.head_dim)
        lse = torch.empty(self.n_heads, max(rows, 1), dtype=torch.float32, device=q.device)
        attention_forward(self.plan, self.schedule, q, k, v, self.ctx, self.program, self.device_program,
                          out=(o, lse))
        if self.remap_method == "pull":
            y = remap_pull(self.layout, self.peer, buf, self.ctx, tables=(self._pull or (None, None))[0])
        else:
            y = remap_push(self.layout, buf[:rows], self.peer, self.ctx)
        return o, lse, y[:self.layout.linear_rows[self.ctx.rank]]

    def backward_layout(self, y):
        """Linear layout -> attention layout (exact inverse of the remap)."""
        if self.peer is None:
            return remap_inverse(self.layout, y, self.ctx)
        r = self.ctx.rank
        if y.data_ptr() != self.peer.buf.data_ptr():
            self.peer.buf[:y.shape[0]].copy_(y)
        if self.remap_method == "pull":
            x = remap_pull(self.layout, self.peer, self.peer.buf, self.ctx, inverse=True,
                           tables=(self._pull or (None, None))[1])
        else:
            x = remap_push(self.layout, self.peer.buf[:self.layout.linear_rows[r]], self.peer, self.ctx,
                           inverse=True)
        return x[:self.layout.attn_rows[r]]
