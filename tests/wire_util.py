"""Transcript replay harness for frame-level ring peers (CPU oracle peer or
GPU TcpRingEngine): feed a recorded predecessor stream, capture what the peer
sends to its successor."""

from __future__ import annotations

import json
import os
import socket
import threading

import numpy as np

from tests.golden.gen import WIRE_CASES, ring_inputs, sha256

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_wire():
    with open(os.path.join(GOLDEN, "wire.json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(GOLDEN, "wire.npz"))


def case_inputs(c):
    bufs = ring_inputs(c["w"], c["n"], np.dtype(c["dtype"]), c["seed"])
    assert sha256(np.concatenate(bufs) if c["n"] else b"") == c["input_sha256"]
    return bufs


def case_params(i):
    w, n, op, quantize, dtype, seed, chunk_bytes = WIRE_CASES[i]
    return dict(w=w, n=n, op=op, quantize=quantize, dtype=dtype, seed=seed, chunk_bytes=chunk_bytes)


def replay(run, rx_stream: bytes, prefix: bytes = b"") -> bytes:
    """run(tx_sock, rx_sock) executes one peer; rx_stream (after prefix) is what
    its predecessor sends. Returns the bytes the peer sent."""
    a, b = socket.socketpair()  # peer tx -> capture
    c, d = socket.socketpair()  # feed -> peer rx
    out = bytearray()

    def reader():
        while True:
            x = b.recv(1 << 16)
            if not x:
                return
            out.extend(x)

    def writer():
        try:
            c.sendall(prefix + rx_stream)
            c.shutdown(socket.SHUT_WR)
        except OSError:
            pass

    tr = threading.Thread(target=reader, daemon=True)
    tw = threading.Thread(target=writer, daemon=True)
    tr.start()
    tw.start()
    try:
        run(a, d)
    finally:
        try:
            a.shutdown(socket.SHUT_WR)
        except OSError:
            pass
        tr.join(30)
        c.close()
        tw.join(30)
        for s in (a, b, d):
            s.close()
    return bytes(out)


def stale_prefix(tag: int, seq_nr: int) -> bytes:
    """Frames of an aborted earlier attempt (seq_nr - 1) that a peer must discard
    (collective.py:343-356)."""
    import struct

    body = struct.pack(">QQIQI", tag, seq_nr - 1, 0, 0, 8) + bytes(range(8))
    meta = struct.pack(">QQIff", tag, seq_nr - 1, 0, 1.0, 2.0)
    return (struct.pack(">IB", len(meta) + 1, 17) + meta + struct.pack(">IB", len(body) + 1, 15) + body)
