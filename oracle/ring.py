"""NumPy restatement of the reference ring all-reduce data plane.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). Paths cited are
relative to ``/root/reference/pkg``.

Two equivalent forms are provided:

* ``ring_allreduce`` replays the reference schedule step by step over
  rank-indexed buffers (``src/churncomm/collective.py:489-567``, mirrored by
  the reference's own ``tests/oracles.py:30-101``).
* ``reduce_chunk`` is the per-chunk closed form: chunk ``c`` is folded in ring
  order ``x_c, x_{c+1}, ..., x_{c-1}`` as ``acc <- local (+) incoming``, with
  a quantize/dequantize round trip of the running partial at every hop when
  quantization is on, plus the owner's final round trip before the gather.
  It lets parity tests stream config-sized inputs chunk by chunk.

Both are pinned against the reference's own outputs in
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import threading
from enum import IntEnum

import numpy as np


class ReduceOp(IntEnum):
    """Wire codes of ``src/churncomm/wire.py:141-145`` (ReduceOpCode)."""

    SUM = 1
    AVG = 2
    MAX = 3
    MIN = 4
    # extension op (north_star), not in the reference: PARITY UNPINNED -- its
    # oracle is this restatement's own definition, np.multiply folded in the
    # reference's ring order exactly like SUM folds with np.add
    PROD = 5


# collective.py:66-71 -- accumulate(local, incoming, out=local)
_ACCUMULATE = {
    ReduceOp.SUM: np.add,
    ReduceOp.AVG: np.add,
    ReduceOp.MAX: np.maximum,
    ReduceOp.MIN: np.minimum,
    ReduceOp.PROD: np.multiply,
}


def chunk_bounds(n: int, w: int) -> list[tuple[int, int]]:
    """collective.py:86-101: first ``n mod w`` ranks get the ceiling share."""
    if w < 1:
        raise ValueError("world_size must be at least 1")
    base, extra = divmod(n, w)
    out = []
    start = 0
    for r in range(w):
        size = base + (1 if r < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def accumulate(op: ReduceOp, local: np.ndarray, incoming: np.ndarray) -> None:
    """collective.py:407 / :416 -- ``local <- local (+) incoming`` in place."""
    _ACCUMULATE[ReduceOp(op)](local, incoming, out=local)


_scratch = threading.local()


def _scratch_f32(n: int) -> np.ndarray:
    buf = getattr(_scratch, "buf", None)
    if buf is None or buf.size < n:
        buf = np.empty(max(n, 65536), dtype=np.float32)
        _scratch.buf = buf
    return buf[:n]


def quantize_chunk(values: np.ndarray, out: np.ndarray) -> tuple[float, float]:
    """collective.py:109-129: per-span min-max affine u8 quantization.

    ``scale = (max - min) / 255f`` (1 when that is 0);
    ``q = u8(clip(rint((x - min) / scale), 0, 255))``. Empty spans give
    ``(0.0, 1.0)``; non-finite values raise ``ValueError``.
    """
    if values.size == 0:
        return 0.0, 1.0
    if not np.all(np.isfinite(values)):
        raise ValueError("non-finite values cannot be quantized")
    mn = values.min()
    scale = (values.max() - mn) / np.float32(255.0)
    if scale == 0:
        scale = np.float32(1.0)
    sc = _scratch_f32(values.size)
    np.subtract(values, mn, out=sc)
    np.divide(sc, scale, out=sc)
    np.rint(sc, out=sc)
    np.clip(sc, 0.0, 255.0, out=sc)
    np.copyto(out[: values.size], sc, casting="unsafe")
    return float(mn), float(scale)


def dequantize_into(codes: np.ndarray, min_val: float, scale: float, out: np.ndarray) -> None:
    """collective.py:132-135: ``out = f32(q) * scale`` (RN) then ``+ min`` (RN)."""
    np.multiply(codes, np.float32(scale), out=out, casting="unsafe")
    np.add(out, np.float32(min_val), out=out)


def finalize_reduction(buf: np.ndarray, op: ReduceOp, w: int) -> None:
    """collective.py:479-482: AVG divides by ``dtype(W)`` (true division)."""
    if ReduceOp(op) is ReduceOp.AVG:
        np.divide(buf, buf.dtype.type(w), out=buf)


def ring_allreduce(
    buffers: list[np.ndarray], op: ReduceOp, quantize: bool = False
) -> list[np.ndarray]:
    """Replay of ``run_all_reduce`` (collective.py:489-567) over W buffers
    given in ring-position order; returns new arrays (inputs untouched).

    W == 1 finalizes only, without quantization (client.py:896-900).
    """
    op = ReduceOp(op)
    w = len(buffers)
    bufs = [np.array(b, copy=True) for b in buffers]
    if w == 1:
        finalize_reduction(bufs[0], op, 1)
        return bufs
    n = bufs[0].size
    bounds = chunk_bounds(n, w)

    # reduce-scatter: run_reduce_stage, collective.py:371-424 / :521-536
    for step in range(w - 1):
        wire = []
        for r in range(w):
            lo, hi = bounds[(r - step) % w]
            span = bufs[r][lo:hi]
            if quantize:
                codes = np.empty(span.size, dtype=np.uint8)
                mn, sc = quantize_chunk(span, codes)
                if step == 0 and span.size:  # collective.py:387-390
                    dequantize_into(codes, mn, sc, span)
                wire.append((codes, mn, sc))
            else:
                wire.append(span.copy())
        for r in range(w):
            lo, hi = bounds[(r - step - 1) % w]
            incoming = wire[(r - 1) % w]
            if quantize:
                codes, mn, sc = incoming
                part = np.empty(codes.size, dtype=np.float32)
                dequantize_into(codes, mn, sc, part)
                accumulate(op, bufs[r][lo:hi], part)
            else:
                accumulate(op, bufs[r][lo:hi], incoming)

    # gather prologue: collective.py:538-551
    current = [(r + 1) % w for r in range(w)]
    wire = []
    for r in range(w):
        lo, hi = bounds[current[r]]
        own = bufs[r][lo:hi]
        if quantize:
            codes = np.empty(own.size, dtype=np.uint8)
            mn, sc = quantize_chunk(own, codes)
            if own.size:
                dequantize_into(codes, mn, sc, own)
            wire.append((codes, mn, sc))
        else:
            wire.append(own.copy())
    # allgather: run_allgather_stage, collective.py:427-470 / :552-565
    for _ in range(w - 1):
        nxt = [None] * w
        for r in range(w):
            inc = (current[r] - 1) % w
            lo, hi = bounds[inc]
            got = wire[(r - 1) % w]
            if quantize:
                codes, mn, sc = got
                dequantize_into(codes, mn, sc, bufs[r][lo:hi])
            else:
                np.copyto(bufs[r][lo:hi], got)
            nxt[r] = got  # forwarded verbatim
            current[r] = inc
        wire = nxt

    for b in bufs:  # collective.py:567
        finalize_reduction(b, op, w)
    return bufs


def reduce_chunk(spans: list[np.ndarray], op: ReduceOp, quantize: bool, w: int) -> np.ndarray:
    """Closed form of the final value of one chunk.

    ``spans[k]`` is the chunk's slice of the input of ring position
    ``c + k`` (k = 0..W-1), i.e. the fold order of the reference schedule
    (collective.py:522-523: rank r sends chunk (r-step) and receives chunk
    (r-step-1), so chunk c starts at rank c and ends at its owner c-1).
    Equivalent to ``ring_allreduce`` for W >= 2 (checked in tests).
    """
    op = ReduceOp(op)
    acc = np.array(spans[0], copy=True)
    for k in range(1, w):
        if quantize:
            codes = np.empty(acc.size, dtype=np.uint8)
            mn, sc = quantize_chunk(acc, codes)
            dequantize_into(codes, mn, sc, acc)
        local = np.array(spans[k], copy=True)
        accumulate(op, local, acc)
        acc = local
    if quantize and acc.size:
        codes = np.empty(acc.size, dtype=np.uint8)
        mn, sc = quantize_chunk(acc, codes)
        dequantize_into(codes, mn, sc, acc)
    finalize_reduction(acc, op, w)
    return acc


def ring_allreduce_chunkwise(
    buffers: list[np.ndarray], op: ReduceOp, quantize: bool = False
) -> np.ndarray:
    """All-reduce result (identical on every rank) via ``reduce_chunk``."""
    w = len(buffers)
    if w == 1:
        out = np.array(buffers[0], copy=True)
        finalize_reduction(out, op, 1)
        return out
    n = buffers[0].size
    out = np.empty_like(buffers[0])
    for c, (lo, hi) in enumerate(chunk_bounds(n, w)):
        spans = [buffers[(c + k) % w][lo:hi] for k in range(w)]
        out[lo:hi] = reduce_chunk(spans, op, quantize, w)
    return out
