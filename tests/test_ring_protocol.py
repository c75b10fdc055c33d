"""The ring KV pull protocol (program.RingHop, executed by engine._ring_steps
with zp_ring_hop) simulated on the CPU with one compute and one comm thread
per rank, shared "device memory" and epoch flags with the wrap-around
``>=`` wait of the stream memory operations.

Every buffer slot carries a tag (ring, source position) instead of KV rows.
Each round checks that its buffer holds the set of position (i - r) mod g
(reference attention_engine.py:237), each hop checks that the predecessor's
buffer still holds the set it is pulling (no overwrite before the read), and
every wait must complete (no deadlock) — over the reference plans of random
single-box batches, with random delays on both threads of every rank.
"""
import random
import threading

import pytest

from paper_2509_21841_b200 import plan as P, schedule as S
from paper_2509_21841_b200.batch import SequenceBatch
from paper_2509_21841_b200.cluster import ClusterSpec
from paper_2509_21841_b200.program import build_rank_program
from paper_2509_21841_b200.schedule import ring_source

TIMEOUT = 20.0


class Flags:
    """All ranks' flag blocks ("device memory"); wait = stream wait GEQ."""

    def __init__(self, world):
        self.world = world
        self.v = [[0] * (4 * world) for _ in range(world)]  # as engine.RingTransport.flags
        self.cv = threading.Condition()

    def write(self, owner, idx, val):
        with self.cv:
            # a flag only grows (waits compare with >=): a smaller epoch landing
            # after a larger one would strand its waiter
            assert ((val - self.v[owner][idx]) & 0xFFFFFFFF) < 0x80000000, (owner, idx, self.v[owner][idx], val)
            self.v[owner][idx] = val
            self.cv.notify_all()

    def wait(self, owner, idx, val):
        with self.cv:
            ok = self.cv.wait_for(lambda: ((self.v[owner][idx] - val) & 0xFFFFFFFF) < 0x80000000, TIMEOUT)
        if not ok:
            raise TimeoutError(f"flag[{owner}][{idx}] never reached {val}")


def _jitter(rng, scale):
    import time
    time.sleep(rng.random() * scale)


ITERATIONS = 3


def _run_rank(rank, progs, flags, bufs, errors, seed, n_rings):
    """Mirror of engine.attention_steps/_ring_steps for one rank: the comm
    thread runs the hops, the compute thread the pack and rounds; events
    are threading.Events (stream event edges)."""
    rng = random.Random(seed * 131 + rank)
    # per-rank speeds: some ranks' hops lag far behind their rounds and vice versa
    comm_scale, compute_scale = rng.choice([0.0, 0.006]), rng.choice([0.0, 0.006])
    prog = progs[rank]
    world = flags.world
    epoch = 16
    try:
        for it in range(ITERATIONS):
            _one_call(rank, prog, flags, bufs, rng, comm_scale, compute_scale, epoch + it * 16 * n_rings)
    except BaseException as exc:  # noqa: BLE001
        errors.append((rank, exc))


def _one_call(rank, prog, flags, bufs, rng, comm_scale, compute_scale, epoch):
    """One attention_forward: every ring of this rank in schedule order."""
    world = flags.world
    for rp in prog.rings:
        e0 = epoch + 16 * rp.ring_index
        g, me, pred, succ = rp.group_size, rank, rp.prev_rank, rp.next_rank
        nb = rp.n_buffers
        hops = rp.hops()
        ready = {r: threading.Event() for r in range(1, g)}
        done = {r: threading.Event() for r in range(g)}
        comm_err = []

        def comm():
            try:
                for h in hops:
                    if h.free is not None:
                        assert done[h.free].wait(TIMEOUT), "local reader never finished"
                    flags.wait(me, pred, e0 + h.full)
                    if h.free is not None:
                        flags.wait(me, world + succ, e0 + h.free)
                    _jitter(rng, comm_scale)
                    want = (rp.ring_index, (rp.position - 1 - h.round_index) % g)
                    got = bufs[pred][h.src_buf]
                    assert got == want, f"rank {me} hop {h.round_index}: pred buffer holds {got}, want {want}"
                    bufs[me][h.dst_buf] = got
                    flags.write(pred, world + me, e0 + h.consumed)
                    if h.next_full is not None:
                        flags.write(succ, me, e0 + h.next_full)
                    ready[h.round_index + 1].set()
            except BaseException as exc:  # noqa: BLE001
                comm_err.append(exc)

        # compute stream: the previous ring's end wait happened below; pack,
        # then the comm stream starts this ring's hops (event edge)
        bufs[me][0] = (rp.ring_index, rp.position)
        flags.write(succ, me, e0)
        t = threading.Thread(target=comm)
        t.start()
        for r in range(g):
            if r > 0:
                assert ready[r].wait(TIMEOUT), f"rank {me} ring {rp.ring_index}: set for round {r} never came"
            _jitter(rng, compute_scale)
            want = (rp.ring_index, ring_source(rp.position, r, g))
            got = bufs[me][r % nb]
            assert got == want, f"rank {me} round {r}: buffer holds {got}, want {want}"
            done[r].set()
        t.join(TIMEOUT)
        if comm_err:
            raise comm_err[0]
        flags.wait(me, world + succ, e0 + g - 2)


@pytest.mark.parametrize("seed", range(16))
def test_pull_protocol_delivers_every_round_without_races(seed):
    rng = random.Random(seed)
    g = [2, 3, 4, 5, 8, 8, 6, 4][seed % 8]
    lengths = [rng.randint(1, 4000) for _ in range(rng.randint(2, 10))]
    lengths.append(2 * sum(lengths) + rng.randint(2000, 9000))  # > capacity: forces a ring
    total = sum(lengths)
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), ClusterSpec(1, g, -(-total * 105 // (100 * g)),
                                                                               1.0, 1.0))
    sched = S.build_schedule(plan)
    progs = [build_rank_program(plan, sched, r, 4) for r in range(g)]
    flags = Flags(g)
    bufs = [[None] * 3 for _ in range(g)]
    errors = []
    threads = [threading.Thread(target=_run_rank, args=(r, progs, flags, bufs, errors, seed,
                                                                 len(sched.rings()))) for r in range(g)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(4 * TIMEOUT)
    assert not errors, errors
    assert plan.ring_groups


def test_hop_plan_shapes():
    """RingHop fields for a 4-ring: triple buffers, the free wait starts at
    hop 2, the last hop announces nothing onward."""
    lengths = [20000, 100, 200]
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), ClusterSpec(1, 4, 5300, 1.0, 1.0))
    sched = S.build_schedule(plan)
    rp = next(rp for r in range(4) for rp in build_rank_program(plan, sched, r, 4).rings if rp.group_size == 4)
    hops = rp.hops()
    assert rp.n_buffers == 3 and len(hops) == 3
    assert [h.src_buf for h in hops] == [0, 1, 2] and [h.dst_buf for h in hops] == [1, 2, 0]
    assert [h.free for h in hops] == [None, None, 0]
    assert [h.next_full for h in hops] == [1, 2, None]
    assert [h.rows for h in hops] == [rp.recv_rows(r) for r in range(3)]


def _bwd_call(rank, prog, flags, kv, grad, rng, comm_scale, compute_scale, epoch):
    """One attention_backward (engine._ring_bwd_steps): KV sets travel as in
    the forward; each round's dK/dV share is added to the running total pulled
    from the predecessor and announced to the successor; the own set's total
    comes back from the predecessor after the last round.  A partial sum is
    modelled as (ring, set position, frozenset of contributing positions)."""
    world = flags.world
    ng = 3
    for rp in prog.rings:
        e0 = epoch + 16 * rp.ring_index
        g, me, pred, succ, i = rp.group_size, rank, rp.prev_rank, rp.next_rank, rp.position
        nb = rp.n_buffers
        hops = rp.hops()
        ready = {r: threading.Event() for r in range(1, g)}
        done = {r: threading.Event() for r in range(g)}
        comm_err = []

        def comm():
            try:
                for r in range(g):
                    if r < g - 1:
                        h = hops[r]
                        if h.free is not None:
                            assert done[h.free].wait(TIMEOUT)
                        flags.wait(me, pred, e0 + h.full)
                        if h.free is not None:
                            flags.wait(me, world + succ, e0 + h.free)
                        _jitter(rng, comm_scale)
                        kv[me][h.dst_buf] = kv[pred][h.src_buf]
                        flags.write(pred, world + me, e0 + h.consumed)
                        if h.next_full is not None:
                            flags.write(succ, me, e0 + h.next_full)
                        ready[r + 1].set()
                    assert done[r].wait(TIMEOUT), "round never finished"
                    if r > 0:
                        flags.wait(me, 2 * world + pred, e0 + r - 1)
                        _jitter(rng, comm_scale)
                        a = grad[pred][(r - 1) % ng]
                        z = grad[me][r % ng]
                        assert a[:2] == z[:2], f"rank {me} round {r}: pulled total of {a[:2]}, holds {z[:2]}"
                        # previous holders of set (i - r) were positions i-1 .. i-r
                        assert a[2] == frozenset((i - t) % g for t in range(1, r + 1)), (me, r, a)
                        flags.write(pred, 3 * world + me, e0 + r - 1)
                        grad[me][r % ng] = (z[0], z[1], z[2] | a[2])
                    flags.write(succ, 2 * world + me, e0 + r)
                flags.wait(me, 2 * world + pred, e0 + g - 1)
                total = grad[pred][(g - 1) % ng]
                assert total == (rp.ring_index, i, frozenset(range(g))), (me, total)
                flags.write(pred, 3 * world + me, e0 + g - 1)
            except BaseException as exc:  # noqa: BLE001
                comm_err.append(exc)

        kv[me][0] = (rp.ring_index, i)
        flags.write(succ, me, e0)
        t = threading.Thread(target=comm)
        t.start()
        for r in range(g):
            if r > 0:
                assert ready[r].wait(TIMEOUT), f"rank {me}: set for round {r} never came"
            held = kv[me][r % nb]
            assert held == (rp.ring_index, ring_source(i, r, g)), (me, r, held)
            if r >= ng:
                flags.wait(me, 3 * world + succ, e0 + r - ng)  # successor pulled T_{r-3}
            _jitter(rng, compute_scale)
            grad[me][r % ng] = (rp.ring_index, ring_source(i, r, g), frozenset([i]))
            done[r].set()
        t.join(TIMEOUT)
        if comm_err:
            raise comm_err[0]
        flags.wait(me, 3 * world + succ, e0 + g - 1)
        flags.wait(me, world + succ, e0 + g - 2)


@pytest.mark.parametrize("seed", range(12))
def test_backward_pull_protocol_returns_every_total(seed):
    """Ring backward protocol: every pulled running total holds exactly the
    shares of the positions that held the set before, and every position gets
    back the sum of all g shares of its own set, over 2 calls per rank."""
    rng0 = random.Random(1000 + seed)
    g = [2, 3, 4, 5, 8, 6][seed % 6]
    lengths = [rng0.randint(1, 4000) for _ in range(rng0.randint(2, 10))]
    lengths.append(2 * sum(lengths) + rng0.randint(2000, 9000))
    total = sum(lengths)
    plan = P.build_plan(SequenceBatch(tuple(enumerate(lengths))), ClusterSpec(1, g, -(-total * 105 // (100 * g)),
                                                                              1.0, 1.0))
    sched = S.build_schedule(plan)
    progs = [build_rank_program(plan, sched, r, 4) for r in range(g)]
    flags = Flags(g)
    kv = [[None] * 3 for _ in range(g)]
    grad = [[None] * 3 for _ in range(g)]
    errors = []
    n_rings = len(sched.rings())

    def run(r):
        rng = random.Random(seed * 77 + r)
        cs, ks = rng.choice([0.0, 0.005]), rng.choice([0.0, 0.005])
        try:
            for it in range(2):
                _bwd_call(r, progs[r], flags, kv, grad, rng, cs, ks, 16 + it * 16 * n_rings)
        except BaseException as exc:  # noqa: BLE001
            errors.append((r, exc))

    threads = [threading.Thread(target=run, args=(r,)) for r in range(g)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(4 * TIMEOUT)
    assert not errors, errors
