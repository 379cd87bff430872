"""GPU TcpRingEngine (off-box ring peer) against the reference's recorded wire
transcripts and the oracle: byte-identical frames, bit-identical results."""

from __future__ import annotations

import socket
import threading

import numpy as np
import pytest
import torch

from oracle import ring as oring
from oracle import simplehash as osh
from oracle import wire_peer
from tests.golden.gen import WIRE_CASES
from tests.wire_util import case_inputs, load_wire, replay, stale_prefix

pytestmark = pytest.mark.gpu

META, NPZ = load_wire()
OPS = {"sum": 1, "avg": 2, "max": 3, "min": 4}


def _engine(tx, rx, rank, world, chunk_bytes):
    from paper_2505_14065_b200.tcp_ring import TcpRingEngine
    from paper_2505_14065_b200.wire import FrameSocket

    return TcpRingEngine(FrameSocket(tx), FrameSocket(rx), rank, world, "cuda:0", chunk_bytes=chunk_bytes)


@pytest.mark.parametrize("i", range(len(WIRE_CASES)))
def test_replay_reference_transcripts(i):
    c = META["cases"][i]
    bufs = case_inputs(c)
    w = c["w"]
    for r in range(w):
        dev = torch.from_numpy(bufs[r].copy()).cuda()
        counters = []

        def run(tx, rx):
            eng = _engine(tx, rx, r, w, c["chunk_bytes"])
            try:
                counters.append(eng.run_all_reduce(dev, OPS[c["op"]], c["quantize"], c["tag"], c["seq_nr"]))
            finally:
                eng.close()

        prefix = stale_prefix(c["tag"], c["seq_nr"]) if w > 1 else b""
        out = replay(run, NPZ[f"c{i}_tx{(r - 1) % w}"].tobytes(), prefix)
        assert out == NPZ[f"c{i}_tx{r}"].tobytes(), (i, r)
        assert list(counters[0]) == c["counters"][r]
        assert osh.simplehash_np(dev.cpu().numpy()) == c["output_hash"], (i, r)


def _ring(w, make_peer):
    socks = [socket.socketpair() for _ in range(w)]  # link r: rank r -> rank r+1
    errs, res = [], [None] * w

    def work(r):
        try:
            res[r] = make_peer(r, socks[r][0], socks[(r - 1) % w][1])
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))
            for s in socks[r]:
                s.close()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(w)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
        assert not t.is_alive()
    for a, b in socks:
        a.close()
        b.close()
    return res, errs


@pytest.mark.parametrize("quantize,op,w,n", [(False, "avg", 3, 3_000_001), (True, "avg", 3, 1_000_003),
                                           (False, "max", 4, 777_777), (True, "sum", 2, 500_000)])
def test_gpu_ring_and_mixed_ring_match_oracle(quantize, op, w, n):
    rng = np.random.default_rng(n)
    xs = [rng.normal(0, 10, n).astype(np.float32) for _ in range(w)]
    want = oring.ring_allreduce([x.copy() for x in xs], oring.ReduceOp(OPS[op]), quantize=quantize)
    for gpu_ranks in (set(range(w)), set(range(w)) - {1}):
        outs = [torch.from_numpy(x.copy()).cuda() if r in gpu_ranks else x.copy() for r, x in enumerate(xs)]

        def peer(r, tx, rx):
            if r in gpu_ranks:
                eng = _engine(tx, rx, r, w, 64 * 1024)
                try:
                    return eng.run_all_reduce(outs[r], OPS[op], quantize, 5, 9)
                finally:
                    eng.close()
            return wire_peer.run_rank(tx, rx, outs[r], OPS[op], quantize, r, w, 64 * 1024, 5, 9)

        res, errs = _ring(w, peer)
        assert not errs, errs
        for r in range(w):
            got = outs[r].cpu().numpy() if r in gpu_ranks else outs[r]
            assert got.tobytes() == want[r].tobytes(), (r, gpu_ranks)
        for r in range(w):  # what rank r sent is what its successor received
            assert res[r][0] == res[(r + 1) % w][1]


def test_truncated_stream_aborts_and_restores():
    from paper_2505_14065_b200.collective import CollectiveAborted

    i = next(k for k, c in enumerate(WIRE_CASES) if c[:4] == (3, 1000, "sum", True))
    c = META["cases"][i]
    x = case_inputs(c)[1]
    for cut in (0.3, 0.8):
        dev = torch.from_numpy(x.copy()).cuda()
        stream = NPZ[f"c{i}_tx0"].tobytes()

        def run(tx, rx):
            eng = _engine(tx, rx, 1, 3, c["chunk_bytes"])
            try:
                with pytest.raises(CollectiveAborted):
                    eng.run_all_reduce(dev, "sum", True, c["tag"], c["seq_nr"])
            finally:
                eng.close()

        replay(run, stream[: int(len(stream) * cut)])
        assert dev.cpu().numpy().tobytes() == x.tobytes()


def test_nonfinite_quantize_aborts_and_restores():
    from paper_2505_14065_b200.collective import CollectiveAborted

    x = np.arange(1000, dtype=np.float32)
    x[10] = np.inf
    dev = torch.from_numpy(x.copy()).cuda()

    def run(tx, rx):
        eng = _engine(tx, rx, 0, 2, 256)
        try:
            with pytest.raises(CollectiveAborted):
                eng.run_all_reduce(dev, "avg", True, 1, 1)
        finally:
            eng.close()

    replay(run, b"")
    assert dev.cpu().numpy().tobytes() == x.tobytes()
