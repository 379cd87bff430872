"""Frame-level CPU peer of the reference ring (one rank, one attempt).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). A NumPy restatement
of one rank of ``src/churncomm/collective.py:489-567`` (run_all_reduce) over
two framed sockets, speaking the frames of ``src/churncomm/wire.py:153-158``
(length + type), ``:800-822`` (ChunkHeader ``>QQIQI``) and ``:842-858``
(QuantMeta ``>QQIff``). Its own codec (plain ``struct``) is deliberately
independent of the product's ``wire.py``. Pinned against the reference's
recorded transcripts in ``tests/test_wire_cpu.py``; used as a foreign peer in
mixed rings with GPU peers in ``tests/test_tcp_ring_gpu.py``.
"""

from __future__ import annotations

import socket
import struct
import threading

import numpy as np

from . import ring as oring

_HDR = struct.Struct(">IB")
_CHUNK = struct.Struct(">QQIQI")
_QM = struct.Struct(">QQIff")
CHUNK_DATA, QUANT_META = 15, 17


def _recv_exact(sock: socket.socket, n: int) -> bytes:
    out = bytearray()
    while len(out) < n:
        d = sock.recv(n - len(out))
        if not d:
            raise ConnectionError("closed")
        out += d
    return bytes(out)


class _Peer:
    def __init__(self, tx, rx, tag, seq, chunk_bytes):
        self.tx, self.rx, self.tag, self.seq, self.cb = tx, rx, tag, seq, chunk_bytes
        self.tx_bytes = self.rx_bytes = 0

    def send_span(self, stage, payload: bytes, meta) -> None:  # collective.py:285-315
        if meta is not None:
            body = _QM.pack(self.tag, self.seq, stage, meta[0], meta[1])
            self.tx.sendall(_HDR.pack(len(body) + 1, QUANT_META) + body)
            self.tx_bytes += 5 + len(body)
        off = idx = 0
        while off < len(payload):
            n = min(self.cb, len(payload) - off)
            body = _CHUNK.pack(self.tag, self.seq, idx, off, n) + payload[off : off + n]
            self.tx.sendall(_HDR.pack(len(body) + 1, CHUNK_DATA) + body)
            self.tx_bytes += 5 + len(body)
            off += n
            idx += 1

    def recv_stage(self, expect: int, want_meta: bool):  # collective.py:318-368
        data, meta = bytearray(), None
        while (want_meta and meta is None) or len(data) < expect:
            length, typ = _HDR.unpack(_recv_exact(self.rx, 5))
            body = _recv_exact(self.rx, length - 1)
            if typ == QUANT_META:
                tag, seq, _stage, mn, sc = _QM.unpack(body)
                if (tag, seq) != (self.tag, self.seq):
                    continue
                meta = (mn, sc)
                self.rx_bytes += 5 + len(body)
                continue
            assert typ == CHUNK_DATA
            tag, seq, _idx, off, n = _CHUNK.unpack_from(body)
            if (tag, seq) != (self.tag, self.seq):
                continue
            assert off == len(data) and n == len(body) - _CHUNK.size
            data += body[_CHUNK.size :]
            self.rx_bytes += 5 + len(body)
        return bytes(data), meta

    def exchange(self, stage, payload, meta, expect, want_meta):
        err = []

        def send():
            try:
                self.send_span(stage, payload, meta)
            except BaseException as e:  # noqa: BLE001
                err.append(e)

        t = threading.Thread(target=send)
        t.start()
        got = self.recv_stage(expect, want_meta)
        t.join()
        if err:
            raise err[0]
        return got


def run_rank(tx: socket.socket, rx: socket.socket, buf: np.ndarray, op, quantize: bool, rank: int,
             world: int, chunk_bytes: int = 256 * 1024, tag: int = 0, seq_nr: int = 1) -> tuple[int, int]:
    """One rank's attempt; ``buf`` is reduced in place. Returns (tx, rx) payload bytes."""
    op = oring.ReduceOp(op)
    p = _Peer(tx, rx, tag, seq_nr, chunk_bytes)
    w, n = world, buf.size
    bounds = oring.chunk_bounds(n, w)
    dt = buf.dtype
    for step in range(w - 1):  # run_reduce_stage, collective.py:371-424
        tlo, thi = bounds[(rank - step) % w]
        rlo, rhi = bounds[(rank - step - 1) % w]
        if quantize:
            codes = np.empty(thi - tlo, np.uint8)
            meta = oring.quantize_chunk(buf[tlo:thi], codes)
            payload = codes.tobytes()
        else:
            meta, payload = None, buf[tlo:thi].tobytes()
        data, got = p.exchange(step, payload, meta, (rhi - rlo) * (1 if quantize else dt.itemsize), quantize)
        if quantize:
            part = np.empty(rhi - rlo, np.float32)
            oring.dequantize_into(np.frombuffer(data, np.uint8), got[0], got[1], part)
        else:
            part = np.frombuffer(data, dt)
        oring.accumulate(op, buf[rlo:rhi], part)
    cur = (rank + 1) % w  # collective.py:538-551
    lo, hi = bounds[cur]
    if quantize:
        codes = np.empty(hi - lo, np.uint8)
        meta = oring.quantize_chunk(buf[lo:hi], codes)
        if hi > lo:
            oring.dequantize_into(codes, meta[0], meta[1], buf[lo:hi])
        wire = codes.tobytes()
    else:
        meta, wire = None, buf[lo:hi].tobytes()
    for step in range(w - 1):  # run_allgather_stage, collective.py:427-470
        inc = (cur - 1) % w
        rlo, rhi = bounds[inc]
        data, got = p.exchange((w - 1) + step, wire, meta, (rhi - rlo) * (1 if quantize else dt.itemsize), quantize)
        if quantize:
            oring.dequantize_into(np.frombuffer(data, np.uint8), got[0], got[1], buf[rlo:rhi])
        else:
            buf[rlo:rhi] = np.frombuffer(data, dt)
        wire, meta, cur = data, got, inc
    oring.finalize_reduction(buf, op, w)
    return p.tx_bytes, p.rx_bytes
