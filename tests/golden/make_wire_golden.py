"""Record the REFERENCE ring's wire transcripts (tests/golden/wire.npz + wire.json).

Run in the dev container (where /root/reference exists):

    python tests/golden/make_wire_golden.py

Every case runs the reference's own engine (churncomm.collective.run_all_reduce
with FrameConn peers, as pkg/tests/ring_harness.py wires them) over
socketpairs, with a relay thread on every ring link that records the exact
bytes each rank sends to its successor. The fixtures hold, per case and rank,
the transmitted byte stream, the payload counters and the simplehash of the
final buffer; the inputs come from tests/golden/gen.py seeds. A rank's
transmitted stream is a function of its input and of the stream it receives,
so replaying rank r-1's transcript into one of our peers must reproduce rank
r's transcript byte for byte (tests/test_tcp_ring_gpu.py). Nothing at test
time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import socket
import sys
import threading

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path[:0] = [REF_SRC]
sys.dont_write_bytecode = True

from churncomm.collective import BufferPool, OpContext, ReduceOp, SpanSender, run_all_reduce  # noqa: E402
from churncomm.sharedstate import simplehash  # noqa: E402
from churncomm.wire import FrameConn  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden.gen import WIRE_CASES, ring_inputs, sha256  # noqa: E402

OPS = {"sum": ReduceOp.SUM, "avg": ReduceOp.AVG, "max": ReduceOp.MAX, "min": ReduceOp.MIN}


def _relay(src: socket.socket, dst: socket.socket, log: bytearray) -> None:
    while True:
        data = src.recv(1 << 16)
        if not data:
            dst.shutdown(socket.SHUT_WR)
            return
        log += data
        dst.sendall(data)


def run_case(w, n, op, quantize, dtype, seed, chunk_bytes, tag, seq):
    bufs = ring_inputs(w, n, np.dtype(dtype), seed)
    inputs_sha = sha256(np.concatenate(bufs) if n else b"")
    logs = [bytearray() for _ in range(w)]
    tx, rx, relays, raw = [None] * w, [None] * w, [], []
    for r in range(w):
        a, b = socket.socketpair()  # rank r -> relay
        c, d = socket.socketpair()  # relay -> rank r+1
        raw += [a, b, c, d]
        tx[r] = FrameConn(a)
        rx[(r + 1) % w] = FrameConn(d)
        t = threading.Thread(target=_relay, args=(b, c, logs[r]), daemon=True)
        t.start()
        relays.append(t)
    results = [None] * w
    counters = [None] * w

    def work(r):
        ctx = OpContext(tag=tag, seq_nr=seq, buffer=bufs[r], op=OPS[op], quantize=quantize, rank=r,
                        world=w, tx_conn=tx[r], rx_conn=rx[r], abort_event=threading.Event(),
                        pool=BufferPool(), chunk_bytes=chunk_bytes)
        sender = SpanSender(f"s{r}")
        try:
            run_all_reduce(ctx, sender)
            results[r] = "ok"
            counters[r] = (ctx.tx_payload_bytes, ctx.rx_payload_bytes)
        finally:
            sender.shutdown()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(w)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(60)
        assert not t.is_alive()
    assert results == ["ok"] * w
    for r in range(w):
        raw[4 * r].shutdown(socket.SHUT_WR)
    for t in relays:
        t.join(10)
    for s in raw:
        s.close()
    hashes = [simplehash(b) for b in bufs]
    assert len(set(hashes)) == 1
    return inputs_sha, [bytes(x) for x in logs], counters, hashes[0]


def main():
    arrays, meta = {}, []
    for i, (w, n, op, quantize, dtype, seed, chunk_bytes) in enumerate(WIRE_CASES):
        tag, seq = 7, 3
        inputs_sha, logs, counters, out_hash = run_case(w, n, op, quantize, dtype, seed, chunk_bytes, tag, seq)
        for r in range(w):
            arrays[f"c{i}_tx{r}"] = np.frombuffer(logs[r], dtype=np.uint8)
        meta.append({"w": w, "n": n, "op": op, "quantize": quantize, "dtype": dtype, "seed": seed,
                     "chunk_bytes": chunk_bytes, "tag": tag, "seq_nr": seq, "input_sha256": inputs_sha,
                     "counters": counters, "output_hash": out_hash,
                     "tx_sha256": [sha256(np.frombuffer(x, np.uint8)) for x in logs]})
    np.savez_compressed(os.path.join(HERE, "wire.npz"), **arrays)
    with open(os.path.join(HERE, "wire.json"), "w") as f:
        json.dump({"cases": meta, "codec": codec_goldens()}, f, indent=1)
    print(f"{len(meta)} wire cases, {sum(a.size for a in arrays.values())} transcript bytes")


def codec_goldens():
    from churncomm import wire

    hdr = wire.ChunkHeader(tag=8, seq_nr=2, chunk_index=5, byte_offset=4096, byte_len=12)
    qm = wire.QuantMeta(8, 2, 1, -1.5, 0.25)
    return {
        "chunk_header": hdr.pack().hex(),
        "quant_meta": qm.pack().hex(),
        "frame_chunk": wire.encode_frame(wire.MessageType.CHUNK_DATA, hdr.pack() + b"abcdefghijkl").hex(),
        "frame_meta": wire.encode_frame(wire.MessageType.QUANT_META, qm.pack()).hex(),
        "frame_empty": wire.encode_frame(wire.MessageType.CHUNK_DATA, b"").hex(),
        "init_vote": wire.CollectiveInitVote(8, 1 << 20, wire.DType.F32, wire.ReduceOpCode.AVG, True).pack().hex(),
        "init_vote_f64": wire.CollectiveInitVote(2**63 + 5, 3, wire.DType.F64, wire.ReduceOpCode.MIN, False).pack().hex(),
        "complete_vote": wire.CollectiveCompleteVote(8, 2, True, 100, 101).pack().hex(),
        "complete_vote_fail": wire.CollectiveCompleteVote(9, 7, False).pack().hex(),
        "init_vote_type": int(wire.MessageType.COLLECTIVE_INIT_VOTE),
        "complete_vote_type": int(wire.MessageType.COLLECTIVE_COMPLETE_VOTE),
        "chunk_data": int(wire.MessageType.CHUNK_DATA),
        "quant_meta_type": int(wire.MessageType.QUANT_META),
    }


if __name__ == "__main__":
    main()
