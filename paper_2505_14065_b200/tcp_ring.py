"""Off-box ring peer: the reference's TCP data-frame protocol, GPU arithmetic.

``TcpRingEngine`` runs one attempt of the reference's pipelined ring
(collective.py:489-567) for a CUDA buffer over a pair of framed TCP
connections (to the ring successor, from the predecessor), byte-compatible
with the reference's ``FrameConn`` peers (wire.py; docs/protocol.md
ChunkData/QuantMeta). It is the transport for peers that are not on the same
NVLink box: the chunk arithmetic stays on the GPU
(accumulate, range, quantize, dequant-accumulate, finalize kernels of
libpcclb200), frames move through pinned host staging, sends run on a sender
thread while the caller thread receives (SpanSender, collective.py:192-230).
Frames of other attempts are discarded as in collective.py:343-356.
"""

from __future__ import annotations

import socket
from concurrent.futures import ThreadPoolExecutor

import torch

from ._native import check, lib
from .collective import DTYPE_CODE, CollectiveAborted, QuantScratch, ReduceOp, UsageError, compute_chunk_boundaries
from .wire import (
    CHUNK_DATA,
    CHUNK_HEADER_LEN,
    FRAME_OVERHEAD,
    QUANT_META,
    QUANT_META_LEN,
    ChunkHeader,
    ConnectionClosed,
    FrameSocket,
    ProtocolError,
    QuantMeta,
)


def _join_quiet(fut) -> None:
    try:
        fut.result()
    except BaseException:
        pass


class TcpRingEngine:
    def __init__(self, tx: FrameSocket, rx: FrameSocket, rank: int, world: int, device=None,
                 chunk_bytes: int = 256 * 1024, recv_timeout: float | None = 60.0):
        self.tx, self.rx = tx, rx
        rx.sock.settimeout(recv_timeout)  # RecvTimeout of collective.py:333
        self.rank, self.world = rank, world
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.chunk_bytes = chunk_bytes
        self.stream = torch.cuda.Stream(self.device)
        self.sender = ThreadPoolExecutor(max_workers=1)
        self.rx_host = [torch.empty(chunk_bytes + CHUNK_HEADER_LEN + 64, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.rx_ev = [torch.cuda.Event() for _ in range(2)]
        self.dev_rx = torch.empty(chunk_bytes, dtype=torch.uint8, device=self.device)
        self.scratch = QuantScratch(self.device)
        self.rx_meta_dev = torch.empty(2, dtype=torch.float32, device=self.device)
        self.rx_meta_host = torch.empty(2, dtype=torch.float32, pin_memory=True)
        self._wire = [torch.empty(0, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
        self.tx_payload_bytes = 0
        self.rx_payload_bytes = 0

    def close(self) -> None:
        self.sender.shutdown(wait=True)

    def _unblock_sender(self) -> None:
        # the reference sets abort_event (collective.py:413-416); a blocked
        # sendmsg is released by shutting the successor connection down
        try:
            self.tx.sock.shutdown(socket.SHUT_RDWR)
        except OSError:
            pass

    # -- host staging -------------------------------------------------------
    def _wire_buf(self, i: int, nbytes: int) -> torch.Tensor:
        if self._wire[i].numel() < nbytes:
            self._wire[i] = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        return self._wire[i][:nbytes]

    def _d2h(self, dev_bytes: torch.Tensor, host: torch.Tensor) -> None:
        with torch.cuda.stream(self.stream):
            host.copy_(dev_bytes, non_blocking=True)
        self.stream.synchronize()

    # -- frames (collective.py:285-368) --------------------------------------
    def _send_span(self, tag, seq, stage, payload: torch.Tensor, meta) -> None:
        if meta is not None:
            body = QuantMeta(tag, seq, stage, meta[0], meta[1]).pack()
            self.tx.send_frame(QUANT_META, body)
            self.tx_payload_bytes += FRAME_OVERHEAD + len(body)
        mv = memoryview(payload.numpy()).cast("B") if payload.numel() else memoryview(b"")
        total, off, idx = len(mv), 0, 0
        while off < total:
            n = min(self.chunk_bytes, total - off)
            self.tx.send_frame(CHUNK_DATA, ChunkHeader(tag, seq, idx, off, n).pack(), mv[off : off + n])
            self.tx_payload_bytes += FRAME_OVERHEAD + CHUNK_HEADER_LEN + n
            off += n
            idx += 1

    def _recv_stage(self, tag, seq, expect: int, want_meta: bool, consume):
        """consume(offset, host_view, slot) is called per data frame."""
        received, meta, k = 0, None, 0
        while (want_meta and meta is None) or received < expect:
            slot = k % 2
            self.rx_ev[slot].synchronize()  # the H2D that read this staging slot is done
            buf = self.rx_host[slot]
            msg_type, length = self.rx.recv_frame_into(buf.numpy())
            view = memoryview(buf.numpy())[:length]
            if msg_type == QUANT_META:
                qm = QuantMeta.unpack(view)
                if (qm.tag, qm.seq_nr) != (tag, seq):
                    continue
                if not want_meta:
                    raise ProtocolError("unexpected quantization metadata")
                meta = (qm.min_val, qm.scale)
                self.rx_payload_bytes += FRAME_OVERHEAD + QUANT_META_LEN
                continue
            if msg_type != CHUNK_DATA:
                raise ProtocolError(f"unexpected message {msg_type} on data connection")
            h = ChunkHeader.unpack_from(view)
            if (h.tag, h.seq_nr) != (tag, seq):
                if h.tag == tag and h.seq_nr > seq:
                    raise ProtocolError("data from a future attempt")
                continue
            if h.byte_offset != received:
                raise ProtocolError("out-of-order chunk within stage")
            if h.byte_offset + h.byte_len > expect:
                raise ProtocolError("chunk exceeds stage span")
            if want_meta and meta is None:
                raise ProtocolError("chunk data arrived before quantization metadata")
            consume(h.byte_offset, buf[CHUNK_HEADER_LEN : CHUNK_HEADER_LEN + h.byte_len], slot, meta)
            received += h.byte_len
            self.rx_payload_bytes += FRAME_OVERHEAD + CHUNK_HEADER_LEN + h.byte_len
            k += 1
        return meta

    # -- GPU steps -----------------------------------------------------------
    def _quantize(self, span: torch.Tensor, host_codes: torch.Tensor, adopt: bool, avg_div: int):
        """Range + quantize on the GPU (collective.py:109-129); codes to host."""
        L = lib()
        s = self.stream.cuda_stream
        n = span.numel()
        codes = torch.empty(max(n, 1), dtype=torch.uint8, device=self.device)
        check(L.pcclb_range_reset(self.scratch.range.data_ptr(), 1, s), "range_reset")
        if n:
            check(L.pcclb_range_f32(span.data_ptr(), n, self.scratch.range.data_ptr(), s), "range")
        check(L.pcclb_quantize_u8(span.data_ptr(), n, self.scratch.range.data_ptr(), codes.data_ptr(),
                                  self.scratch.meta.data_ptr(), span.data_ptr() if adopt else None, avg_div, s),
              "quantize")
        self.stream.synchronize()
        if int(self.scratch.range[2].item()) != 0:
            raise ValueError("non-finite values cannot be quantized")
        if n:
            self._d2h(codes[:n], host_codes)
        m = self.scratch.meta.cpu()
        return float(m[0]), float(m[1])

    def _meta_h2d(self, meta) -> None:
        # the previous stage's kernels finished (stream synchronised per stage)
        self.rx_meta_host[0], self.rx_meta_host[1] = meta
        with torch.cuda.stream(self.stream):
            self.rx_meta_dev.copy_(self.rx_meta_host, non_blocking=True)

    def _h2d(self, host: torch.Tensor, dev: torch.Tensor, slot: int) -> None:
        with torch.cuda.stream(self.stream):
            dev.copy_(host, non_blocking=True)
        self.rx_ev[slot].record(self.stream)

    def run_all_reduce(self, buffer: torch.Tensor, op=ReduceOp.SUM, quantize: bool = False,
                       tag: int = 0, seq_nr: int = 1) -> tuple[int, int]:
        op = ReduceOp.parse(op)
        if op is ReduceOp.PROD:
            raise UsageError("PROD is an extension op (north_star): the reference's TCP peers do not implement it")
        if buffer.dtype == torch.bfloat16:
            raise UsageError("bf16 is an extension dtype: the reference's frames carry f32/f64 (wire.py DType)")
        if quantize not in (False, True, None, "u8"):
            raise UsageError(f"the TCP frames carry u8 min-max codes only (wire.py QuantMeta), not {quantize!r}")
        if not isinstance(buffer, torch.Tensor) or buffer.dim() != 1 or not buffer.is_contiguous() or not buffer.is_cuda:
            raise UsageError("buffer must be a one-dimensional contiguous CUDA tensor")
        if buffer.dtype not in DTYPE_CODE or (quantize and buffer.dtype != torch.float32):
            raise UsageError("unsupported dtype / quantization combination")
        self.tx_payload_bytes = self.rx_payload_bytes = 0
        torch.cuda.current_stream(self.device).synchronize()
        backup = buffer.clone()  # collective.py:501-504
        try:
            self._run(buffer, op, quantize, tag, seq_nr)
        except (ConnectionClosed, ProtocolError, OSError, ValueError) as e:
            self._unblock_sender()
            self.stream.synchronize()
            buffer.copy_(backup)  # collective.py:571-574 (and the non-finite case)
            raise CollectiveAborted(f"io failure: {e}", source="io") from e
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return self.tx_payload_bytes, self.rx_payload_bytes

    def _run(self, buf, op, quantize, tag, seq):
        L = lib()
        s = self.stream.cuda_stream
        w, rank = self.world, self.rank
        n = buf.numel()
        esz = buf.element_size()
        dt = DTYPE_CODE[buf.dtype]
        if w == 1:  # client.py:896-900
            check(L.pcclb_finalize(buf.data_ptr(), n, dt, op.code, 1, s), "finalize")
            self.stream.synchronize()
            return
        bounds = compute_chunk_boundaries(n, w)
        raw = buf.view(torch.uint8)

        def span(c):
            lo, hi = bounds[c]
            return lo, hi

        for step in range(w - 1):  # run_reduce_stage, collective.py:371-424
            tlo, thi = span((rank - step) % w)
            rlo, rhi = span((rank - step - 1) % w)
            if quantize:
                host = self._wire_buf(0, thi - tlo)
                meta = self._quantize(buf[tlo:thi], host, adopt=False, avg_div=1) if thi > tlo else (0.0, 1.0)
            else:
                host = self._wire_buf(0, (thi - tlo) * esz)
                if thi > tlo:
                    self._d2h(raw[tlo * esz : thi * esz], host)
                meta = None
            fut = self.sender.submit(self._send_span, tag, seq, step, host, meta)

            def consume(off, view, slot, m, rlo=rlo):
                nb = view.numel()
                dev = self.dev_rx[:nb]
                self._h2d(view, dev, slot)
                if quantize:
                    if off == 0:
                        self._meta_h2d(m)
                    check(L.pcclb_dequant_accumulate_u8(buf.data_ptr() + (rlo + off) * 4, dev.data_ptr(), nb,
                                                        self.rx_meta_dev.data_ptr(), op.code, None, s), "dq_acc")
                else:
                    if nb % esz:
                        raise ProtocolError("chunk not a whole number of elements")
                    check(L.pcclb_accumulate(buf.data_ptr() + rlo * esz + off, dev.data_ptr(), nb // esz, dt,
                                             op.code, s), "accumulate")

            try:
                self._recv_stage(tag, seq, (rhi - rlo) * (1 if quantize else esz), quantize, consume)
            except BaseException:
                self._unblock_sender()
                _join_quiet(fut)
                raise
            fut.result()
            self.stream.synchronize()

        # gather prologue (collective.py:538-551)
        cur = (rank + 1) % w
        lo, hi = span(cur)
        if quantize:
            wire = self._wire_buf(1, hi - lo)
            meta = self._quantize(buf[lo:hi], wire, adopt=True, avg_div=1) if hi > lo else (0.0, 1.0)
        else:
            wire = self._wire_buf(1, (hi - lo) * esz)
            if hi > lo:
                self._d2h(raw[lo * esz : hi * esz], wire)
            meta = None
        for step in range(w - 1):  # run_allgather_stage, collective.py:427-470
            inc = (cur - 1) % w
            rlo, rhi = span(inc)
            nbytes = (rhi - rlo) * (1 if quantize else esz)
            nxt = self._wire_buf(2 if step % 2 == 0 else 1, nbytes)
            fut = self.sender.submit(self._send_span, tag, seq, (w - 1) + step, wire, meta)

            def consume(off, view, slot, m, nxt=nxt, rlo=rlo):
                nb = view.numel()
                nxt[off : off + nb].copy_(view)  # kept for verbatim forwarding
                if not quantize:
                    if nb % esz:
                        raise ProtocolError("chunk not a whole number of elements")
                    self._h2d(view, raw[rlo * esz + off : rlo * esz + off + nb], slot)

            try:
                got = self._recv_stage(tag, seq, nbytes, quantize, consume)
            except BaseException:
                self._unblock_sender()
                _join_quiet(fut)
                raise
            fut.result()
            if quantize and rhi > rlo:
                codes = self.dev_rx if nbytes <= self.dev_rx.numel() else torch.empty(nbytes, dtype=torch.uint8, device=self.device)
                with torch.cuda.stream(self.stream):
                    codes[:nbytes].copy_(nxt, non_blocking=True)
                self._meta_h2d(got)
                check(L.pcclb_dequantize_u8(buf.data_ptr() + rlo * 4, codes.data_ptr(), rhi - rlo,
                                            self.rx_meta_dev.data_ptr(), 1, s), "dequantize")
            self.stream.synchronize()
            wire, meta = nxt, got
            cur = inc
        check(L.pcclb_finalize(buf.data_ptr(), n, dt, op.code, w, s), "finalize")  # collective.py:567
        self.stream.synchronize()
