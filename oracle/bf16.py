"""bf16 all-reduce definition -- TEST INFRASTRUCTURE ONLY (see
``oracle/__init__.py``). PARITY UNPINNED: the reference reduces f32/f64 only
(collective.py:73-74, wire.py DType), so this NumPy restatement is the
specification: bf16 values are uint16 bit patterns; every fold step of the
reference's ring order computes in float32 with NumPy's ufuncs and rounds the
result to bf16 (round to nearest even, a NaN keeps sign and payload,
quieted); np.maximum/np.minimum select one of the two bf16 operands
unchanged; AVG divides in float32 and rounds.
"""

from __future__ import annotations

import numpy as np

from .ring import ReduceOp, chunk_bounds


def to_f32(u16: np.ndarray) -> np.ndarray:
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def from_f32(f: np.ndarray) -> np.ndarray:
    u = np.asarray(f, dtype=np.float32).view(np.uint32)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    rne = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return np.where(nan, ((u >> 16) | 0x40).astype(np.uint16), rne)


def accumulate(op: ReduceOp, local: np.ndarray, incoming: np.ndarray) -> np.ndarray:
    """local (+) incoming on bf16 bit patterns (returns a new array)."""
    a, b = to_f32(local), to_f32(incoming)
    op = ReduceOp(op)
    with np.errstate(all="ignore"):
        if op == ReduceOp.MAX:
            return np.where((a > b) | np.isnan(a), local, incoming).astype(np.uint16)
        if op == ReduceOp.MIN:
            return np.where((a < b) | np.isnan(a), local, incoming).astype(np.uint16)
        if op == ReduceOp.PROD:
            return from_f32(np.multiply(a, b))
        return from_f32(np.add(a, b))


def ring_allreduce_chunkwise(buffers: list[np.ndarray], op: ReduceOp) -> np.ndarray:
    """Closed form per chunk: chunk c folds positions c, c+1, ..., c-1 as
    acc <- local (+) acc (the reference's order, SURVEY §0 finding 2)."""
    w = len(buffers)
    n = buffers[0].size
    out = np.empty(n, dtype=np.uint16)
    for c, (lo, hi) in enumerate(chunk_bounds(n, w)):
        acc = np.asarray(buffers[c % w][lo:hi], dtype=np.uint16).copy()
        for k in range(1, w):
            acc = accumulate(op, buffers[(c + k) % w][lo:hi], acc)
        if ReduceOp(op) == ReduceOp.AVG:
            with np.errstate(all="ignore"):
                acc = from_f32(to_f32(acc) / np.float32(w))
        out[lo:hi] = acc
    return out
