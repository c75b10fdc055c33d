"""Measured timelines in the reference's Chrome-trace schema.

The reference exports *modelled* timelines (simulator.py:365-382): complete
("X") events, microsecond timestamps, pid = node, tid = "rank.stream" with
streams compute / intra-comm / inter-comm, and event kinds
``{ring.kind}.attn``, ``kv.send``, ``local.attn``, ``kv.allgather``,
``remap.forward`` / ``remap.inverse``, ``linear``.  A ``Tracer`` attached to a
``RankContext`` records CUDA events around the same operations as they run
on the GPUs, and ``export`` writes the measured timeline of every rank in that
schema, so modelled and measured runs load side by side in Perfetto.
"""

from __future__ import annotations

import contextlib
import json

import torch

COMPUTE, INTRA_COMM, INTER_COMM = "compute", "intra-comm", "inter-comm"


class Tracer:
    def __init__(self, device=None):
        self.device = device
        self.base = torch.cuda.Event(enable_timing=True)
        self.base.record()
        self.records: list[tuple[str, str, dict, torch.cuda.Event, torch.cuda.Event]] = []

    @contextlib.contextmanager
    def span(self, stream_name: str, kind: str, payload: dict | None = None, stream=None):
        s = stream or torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        try:
            yield
        finally:
            b.record(s)
            self.records.append((stream_name, kind, dict(payload or {}), a, b))

    def events(self, rank: int) -> list[dict]:
        """(rank, stream, start s, duration s, kind, payload) after a sync."""
        torch.cuda.synchronize()
        out = []
        for stream, kind, payload, a, b in self.records:
            start = self.base.elapsed_time(a) / 1e3
            out.append({"rank": rank, "stream": stream, "start": start,
                        "duration": max(a.elapsed_time(b), 0.0) / 1e3, "kind": kind, "payload": payload})
        return out


_ORDER = {COMPUTE: 0, INTRA_COMM: 1, INTER_COMM: 2}


def to_chrome(events: list[dict], gpus_per_node: int) -> dict:
    recs = []
    for e in sorted(events, key=lambda e: (e["start"], e["rank"], _ORDER.get(e["stream"], 9), e["kind"],
                                           e["duration"])):
        recs.append({"name": e["kind"], "ph": "X", "ts": e["start"] * 1e6, "dur": e["duration"] * 1e6,
                     "pid": e["rank"] // gpus_per_node, "tid": f"{e['rank']}.{e['stream']}",
                     "args": {k: v for k, v in sorted(e["payload"].items())}})
    return {"displayTimeUnit": "ms", "traceEvents": recs}


def export(tracer: Tracer, ctx, path: str, gpus_per_node: int | None = None) -> dict | None:
    """Gather every rank's events (collective when world > 1) and write the
    trace on rank 0.  Returns the trace dict on rank 0."""
    evs = tracer.events(ctx.rank)
    if ctx.world > 1:
        import torch.distributed as dist
        everyone = [None] * ctx.world
        dist.all_gather_object(everyone, evs, group=ctx.group)
        evs = [e for part in everyone for e in part]
    if ctx.rank != 0:
        return None
    doc = to_chrome(evs, gpus_per_node or ctx.world)
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")
    return doc
