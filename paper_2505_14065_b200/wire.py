"""Off-box data frames of the ring, byte-compatible with the reference.

The reference's framing (docs/protocol.md:1-40, :170-203; wire.py:153-176,
:796-862): every frame is a 4-byte big-endian length (type byte + payload),
one type byte, then the payload. A ring stage is an optional QUANT_META frame
``>QQIff`` (tag, seq_nr, stage, min f32, scale f32) followed by CHUNK_DATA
frames whose payload is a 32-byte ``>QQIQI`` header (tag, seq_nr,
chunk_index, byte_offset, byte_len) and up to ``chunk_bytes`` raw
little-endian element (or u8 code) bytes.
"""

from __future__ import annotations

import socket
import struct
from dataclasses import dataclass

COLLECTIVE_INIT_VOTE = 13  # MessageType (wire.py:71)
COLLECTIVE_COMPLETE_VOTE = 14  # MessageType (wire.py:72)
CHUNK_DATA = 15  # MessageType.CHUNK_DATA (wire.py:73)
QUANT_META = 17  # MessageType.QUANT_META (wire.py:75)

_FRAME = struct.Struct(">IB")
_CHUNK = struct.Struct(">QQIQI")
_QMETA = struct.Struct(">QQIff")
_INIT = struct.Struct(">QQBBB")
_COMPLETE = struct.Struct(">QQBQQ")
FRAME_OVERHEAD = _FRAME.size  # 5
CHUNK_HEADER_LEN = _CHUNK.size  # 32
QUANT_META_LEN = _QMETA.size  # 28
MAX_PAYLOAD = (1 << 32) - 2


class ProtocolError(Exception):
    pass


class ConnectionClosed(Exception):
    pass


@dataclass
class ChunkHeader:
    tag: int
    seq_nr: int
    chunk_index: int
    byte_offset: int
    byte_len: int

    def pack(self) -> bytes:
        return _CHUNK.pack(self.tag, self.seq_nr, self.chunk_index, self.byte_offset, self.byte_len)

    @classmethod
    def unpack_from(cls, buf, offset: int = 0) -> "ChunkHeader":
        return cls(*_CHUNK.unpack_from(buf, offset))


@dataclass
class QuantMeta:
    tag: int
    seq_nr: int
    stage: int
    min_val: float
    scale: float

    def pack(self) -> bytes:
        return _QMETA.pack(self.tag, self.seq_nr, self.stage, self.min_val, self.scale)

    @classmethod
    def unpack(cls, buf) -> "QuantMeta":
        if len(buf) != QUANT_META_LEN:
            raise ProtocolError("bad QuantMeta length")
        return cls(*_QMETA.unpack(bytes(buf)))


@dataclass
class CollectiveInitVote:
    """wire.py:754-773: the op descriptor every peer votes on before an
    attempt (dtype 1 f32 / 2 f64, op 1..4 as ReduceOpCode)."""

    tag: int
    element_count: int
    dtype: int
    op: int
    quantize: bool

    def pack(self) -> bytes:
        return _INIT.pack(self.tag, self.element_count, self.dtype, self.op, 1 if self.quantize else 0)

    @classmethod
    def unpack(cls, buf) -> "CollectiveInitVote":
        if len(buf) != _INIT.size:
            raise ProtocolError("bad CollectiveInitVote length")
        tag, count, dtype, op, quant = _INIT.unpack(bytes(buf))
        return cls(tag, count, dtype, op, bool(quant))


@dataclass
class CollectiveCompleteVote:
    """wire.py:776-794: outcome vote with the attempt's payload counters."""

    tag: int
    seq_nr: int
    ok: bool
    tx_bytes: int = 0
    rx_bytes: int = 0

    def pack(self) -> bytes:
        return _COMPLETE.pack(self.tag, self.seq_nr, 1 if self.ok else 0, self.tx_bytes, self.rx_bytes)

    @classmethod
    def unpack(cls, buf) -> "CollectiveCompleteVote":
        if len(buf) != _COMPLETE.size:
            raise ProtocolError("bad CollectiveCompleteVote length")
        tag, seq, ok, tx, rx = _COMPLETE.unpack(bytes(buf))
        return cls(tag, seq, bool(ok), tx, rx)


def frame_header(msg_type: int, payload_len: int) -> bytes:
    if payload_len > MAX_PAYLOAD:
        raise ProtocolError("payload exceeds frame limit")
    return _FRAME.pack(payload_len + 1, msg_type)


def encode_frame(msg_type: int, payload: bytes = b"") -> bytes:
    return frame_header(msg_type, len(payload)) + bytes(payload)


class FrameSocket:
    """Blocking framed socket: scatter-send a frame without copying the
    payload, receive a frame into a caller buffer."""

    def __init__(self, sock: socket.socket):
        self.sock = sock

    def send_frame(self, msg_type: int, *parts) -> None:
        total = sum(len(p) for p in parts)
        bufs = [frame_header(msg_type, total), *[memoryview(p).cast("B") for p in parts]]
        while bufs:
            sent = self.sock.sendmsg(bufs)
            while bufs and sent >= len(bufs[0]):
                sent -= len(bufs[0])
                bufs.pop(0)
            if bufs and sent:
                bufs[0] = bufs[0][sent:]

    def _recv_exact(self, view: memoryview) -> None:
        got = 0
        while got < len(view):
            n = self.sock.recv_into(view[got:])
            if n == 0:
                raise ConnectionClosed("peer closed the data connection")
            got += n

    def recv_frame_into(self, buf) -> tuple[int, int]:
        """Read one frame's payload into buf; returns (type, payload length)."""
        hdr = bytearray(FRAME_OVERHEAD)
        self._recv_exact(memoryview(hdr))
        length, msg_type = _FRAME.unpack(hdr)
        if length < 1:
            raise ProtocolError("frame length below 1")
        n = length - 1
        view = memoryview(buf).cast("B")
        if n > len(view):
            raise ProtocolError("frame larger than the receive buffer")
        self._recv_exact(view[:n])
        return msg_type, n

    def close(self) -> None:
        self.sock.close()
