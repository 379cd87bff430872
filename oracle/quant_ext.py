"""Quantization formats beyond the reference's u8 min-max -- TEST
INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). PARITY UNPINNED: the
reference has no u16 or zero-point quantization, so these
NumPy definitions are the specification the GPU kernels are checked against.
They follow ``quantize_chunk`` / ``dequantize_into`` (collective.py:109-135,
restated in oracle/ring.py) operation by operation in float32:

  u16      scale = (max - min) / 65535 (1 if 0); q = u16(clip(rint((x - min) / scale), 0, 65535))
           D(q) = f32(q) * scale + min
  u8_zp    min/max widened to include 0; scale = (max - min) / 255 (1 if 0);
  u16_zp   zp = clip(rint(-min / scale), 0, L); q = clip(rint(x / scale) + zp, 0, L)
           D(q) = (f32(q) - zp) * scale
NaN -> code 0; every operation rounds once (no FMA).
"""

from __future__ import annotations

import numpy as np

from .ring import ReduceOp, accumulate, chunk_bounds, finalize_reduction

FORMATS = {"u16": (65535, np.uint16, False), "u8_zp": (255, np.uint8, True), "u16_zp": (65535, np.uint16, True)}


def quantize_ex(values: np.ndarray, fmt: str) -> tuple[np.ndarray, float, float]:
    """(codes, p0, scale): p0 is the minimum (min-max) or the zero point."""
    levels, ctype, zp_fmt = FORMATS[fmt]
    values = np.asarray(values, dtype=np.float32)
    if values.size == 0:
        return np.empty(0, ctype), 0.0, 1.0
    mn, mx = np.float32(values.min()), np.float32(values.max())
    if not (np.isfinite(mn) and np.isfinite(mx)):
        raise ValueError("non-finite values cannot be quantized")
    if zp_fmt:
        mn, mx = np.minimum(mn, np.float32(0)), np.maximum(mx, np.float32(0))
    scale = np.float32(np.float32(mx - mn) / np.float32(levels))
    if scale == 0:
        scale = np.float32(1.0)
    with np.errstate(invalid="ignore", over="ignore"):
        if zp_fmt:
            zp = np.float32(np.clip(np.rint(np.float32(-mn) / scale), 0, levels))
            t = np.rint(values / scale) + zp
            p0 = zp
        else:
            t = np.rint((values - mn) / scale)
            p0 = mn
        t = np.clip(t, 0, levels)
        t[np.isnan(t)] = 0
    return t.astype(ctype), float(p0), float(scale)


def dequantize_ex(codes: np.ndarray, p0: float, scale: float, fmt: str) -> np.ndarray:
    _, _, zp_fmt = FORMATS[fmt]
    c = codes.astype(np.float32)
    if zp_fmt:
        return (c - np.float32(p0)) * np.float32(scale)
    return c * np.float32(scale) + np.float32(p0)


def roundtrip(values: np.ndarray, fmt: str) -> np.ndarray:
    codes, p0, scale = quantize_ex(values, fmt)
    return dequantize_ex(codes, p0, scale, fmt)


def reduce_chunk_ex(spans: list[np.ndarray], op: ReduceOp, fmt: str, w: int) -> np.ndarray:
    """oracle.ring.reduce_chunk with the format's quantize/dequantize round trip."""
    acc = np.array(spans[0], dtype=np.float32, copy=True)
    for k in range(1, w):
        acc = roundtrip(acc, fmt)
        local = np.array(spans[k], dtype=np.float32, copy=True)
        accumulate(op, local, acc)
        acc = local
    if acc.size:
        acc = roundtrip(acc, fmt)
    finalize_reduction(acc, op, w)
    return acc


def ring_allreduce_chunkwise_ex(buffers: list[np.ndarray], op: ReduceOp, fmt: str) -> np.ndarray:
    w = len(buffers)
    n = buffers[0].size
    out = np.empty(n, dtype=np.float32)
    if w == 1:  # W = 1: finalize only, never quantized (client.py:896-900)
        out[:] = buffers[0]
        finalize_reduction(out, op, 1)
        return out
    for c, (lo, hi) in enumerate(chunk_bounds(n, w)):
        out[lo:hi] = reduce_chunk_ex([buffers[(c + k) % w][lo:hi] for k in range(w)], op, fmt, w)
    return out
