"""Host-side logic of the NVLink engine on CPU: the schedule executed by W
gloo processes (world_size 2 and 3) with the oracle's arithmetic reproduces
the reference ring result, and the IPC-handle exchange delivers every
rank's handle in ring order. No GPU."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ring as oring
from paper_2505_14065_b200 import schedule


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _simulate(rank, world, port, ring_order, quant, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_14065_b200.ring_ipc import exchange_bytes

        pos = ring_order.index(rank)
        n = 1031
        inputs = [np.random.default_rng(40 + p).normal(0, 3, n).astype(np.float32) for p in range(world)]
        mine = inputs[pos].copy()
        # "workspace" exchange: every rank publishes its input copy (the IPC
        # handle exchange moves handles; here the bytes stand in for memory)
        blobs = exchange_bytes(mine.tobytes())
        peer_in = {ring_order.index(g): np.frombuffer(b, np.float32) for g, b in enumerate(blobs)}
        bounds = oring.chunk_bounds(n, world)
        op = oring.ReduceOp.AVG
        if not quant:
            c = schedule.owned_chunk(pos, world)
            lo, hi = bounds[c]
            acc = peer_in[schedule.fold_chain(pos, world)[0]][lo:hi].copy()
            for p in schedule.fold_chain(pos, world)[1:]:
                local = peer_in[p][lo:hi].copy()
                oring.accumulate(op, local, acc)
                acc = local
            oring.finalize_reduction(acc, op, world)
            res = exchange_bytes(acc.tobytes())
            owned = {schedule.owned_chunk(ring_order.index(g), world): np.frombuffer(b, np.float32) for g, b in enumerate(res)}
            out = mine.copy()
            for chunk, owner in schedule.gather_sources(pos, world) + [(c, pos)]:
                lo2, hi2 = bounds[chunk]
                out[lo2:hi2] = owned[chunk]
        else:
            buf = mine.copy()
            for tx, rx in schedule.quant_steps(pos, world):
                lo, hi = bounds[tx]
                codes = np.empty(hi - lo, np.uint8)
                mn, sc = oring.quantize_chunk(buf[lo:hi], codes)
                got = exchange_bytes(codes.tobytes() + np.array([mn, sc], np.float64).tobytes())
                pred_g = ring_order[(pos - 1) % world]
                blob = got[pred_g]
                pc = np.frombuffer(blob[:-16], np.uint8)
                pmn, psc = np.frombuffer(blob[-16:], np.float64)
                part = np.empty(pc.size, np.float32)
                oring.dequantize_into(pc, float(pmn), float(psc), part)
                lo, hi = bounds[rx]
                oring.accumulate(op, buf[lo:hi], part)
            c = schedule.owned_chunk(pos, world)
            lo, hi = bounds[c]
            codes = np.empty(hi - lo, np.uint8)
            mn, sc = oring.quantize_chunk(buf[lo:hi], codes)
            got = exchange_bytes(codes.tobytes() + np.array([mn, sc], np.float64).tobytes())
            out = buf
            for g, blob in enumerate(got):
                ch = schedule.owned_chunk(ring_order.index(g), world)
                lo, hi = bounds[ch]
                oring.dequantize_into(np.frombuffer(blob[:-16], np.uint8), *np.frombuffer(blob[-16:], np.float64), out[lo:hi])
            oring.finalize_reduction(out, op, world)
        want = oring.ring_allreduce(inputs, op, quantize=quant)[pos]
        q.put((rank, out.tobytes() == want.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("quant", [False, True])
@pytest.mark.parametrize("reverse", [False, True])
def test_schedule_reproduces_reference_gloo(world, quant, reverse):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    order = list(range(world))[::-1] if reverse else list(range(world))
    port = _free_port()
    procs = [ctx.Process(target=_simulate, args=(r, world, port, order, quant, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(results.values()), results


def test_schedule_shapes():
    w = 5
    for pos in range(w):
        chain = schedule.fold_chain(pos, w)
        assert chain[-1] == pos  # the owner folds its own input last (collective.py:407)
        assert sorted(chain) == list(range(w))
        srcs = schedule.gather_sources(pos, w)
        assert len(srcs) == w - 1 and all(schedule.owned_chunk(o, w) == c for c, o in srcs)
    # traffic identity: 2(W-1)/W * N * elem within 1% (test_ring_engine.py:99-108)
    n = 16384
    for w in (2, 3, 6):
        for pos in range(w):
            assert schedule.payload_bytes(n, w, 4, pos) == pytest.approx(2 * (w - 1) / w * n * 4, rel=0.01)


def test_select_sync_plan_rules():
    """master.select_sync_plan rules (master.py:909-976), test_master_units.py:59-147 shape."""
    from paper_2505_14065_b200.communicator import SyncStrategy, select_sync_plan

    E = SyncStrategy.ENFORCE_POPULAR
    # popular hash wins at the top revision; the drifted peer fetches
    reps = {0: (E, [("w", 7, 11, 4)]), 1: (E, [("w", 7, 22, 4)]), 2: (E, [("w", 7, 11, 4)])}
    assert select_sync_plan(reps) == {0: [], 1: [("w", 0, 7, 11)], 2: []}
    # a higher revision beats popularity
    reps = {0: (E, [("w", 3, 11, 4)]), 1: (E, [("w", 9, 22, 4)]), 2: (E, [("w", 3, 11, 4)])}
    assert select_sync_plan(reps) == {0: [("w", 1, 9, 22)], 1: [], 2: [("w", 1, 9, 22)]}
    # tie: smallest hash, then smallest peer
    reps = {0: (E, [("w", 1, 30, 4)]), 1: (E, [("w", 1, 20, 4)]), 2: (E, [("w", 1, 20, 4)]), 3: (E, [("w", 1, 30, 4)])}
    assert select_sync_plan(reps)[0] == [("w", 1, 1, 20)]
    # send-only peers donate even in the minority; receive-only never donate
    S, R = SyncStrategy.SEND_ONLY, SyncStrategy.RECEIVE_ONLY
    reps = {0: (S, [("w", 1, 5, 4)]), 1: (E, [("w", 1, 6, 4)]), 2: (E, [("w", 1, 6, 4)])}
    assert select_sync_plan(reps) == {0: [], 1: [("w", 0, 1, 5)], 2: [("w", 0, 1, 5)]}
    reps = {0: (R, [("w", 1, 5, 4)]), 1: (R, [("w", 1, 6, 4)])}
    assert isinstance(select_sync_plan(reps), str)
