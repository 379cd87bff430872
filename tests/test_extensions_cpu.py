"""CPU checks of the extension oracles (parity unpinned; oracle/quant_ext.py,
oracle/bf16.py): known values and properties their definitions promise."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import bf16 as ob
from oracle import quant_ext as oq
from oracle import ring as oring


def test_bf16_rounding_known_values():
    f = np.array([1.0, -2.5, 1.00390625, 1.005859375, 3.4e38, np.inf, -0.0, 1e-45], np.float32)
    # 1 + 2^-8 is a tie -> even (1.0); 1 + 1.5 * 2^-8 rounds up
    assert ob.from_f32(f).tolist() == [0x3F80, 0xC020, 0x3F80, 0x3F81, 0x7F80, 0x7F80, 0x8000, 0x0000]
    nan = np.array([0x7FA00000], np.uint32).view(np.float32)  # signalling NaN
    assert ob.from_f32(nan)[0] == 0x7FE0  # quieted, payload kept
    assert np.array_equal(ob.to_f32(ob.from_f32(np.float32([0.15625]))), np.float32([0.15625]))


def test_bf16_max_selects_operands():
    a = ob.from_f32(np.float32([1.0, 2.0, -1.0]))
    b = ob.from_f32(np.float32([1.0, 1.0, 5.0]))
    b[0] = 0x3F80
    out = ob.accumulate(oring.ReduceOp.MAX, a, b)
    assert out.tolist() == [b[0], a[1], b[2]]


@pytest.mark.parametrize("fmt", ["u16", "u8_zp", "u16_zp"])
def test_qformat_roundtrip_properties(fmt):
    rng = np.random.default_rng(1)
    x = rng.normal(0.5, 2, 10_000).astype(np.float32)
    codes, p0, scale = oq.quantize_ex(x, fmt)
    levels = oq.FORMATS[fmt][0]
    assert codes.min() >= 0 and codes.max() <= levels
    d = oq.dequantize_ex(codes, p0, scale, fmt)
    assert np.max(np.abs(d - x)) <= scale * 0.5001 + 4e-7 * np.max(np.abs(x))  # half a step + f32 rounding
    if fmt.endswith("_zp"):
        # the zero point encodes 0 exactly
        zero = oq.dequantize_ex(np.array([p0], codes.dtype), p0, scale, fmt)
        assert zero[0] == 0.0
    u8 = np.max(np.abs(oq.roundtrip(x, "u8_zp") - x))
    u16 = np.max(np.abs(oq.roundtrip(x, "u16_zp") - x))
    assert u16 < u8 / 100


def test_qformat_positive_span_keeps_full_range_with_zero_point():
    x = np.float32([3.0, 4.0, 5.0])
    d = oq.roundtrip(x, "u8_zp")
    assert np.max(np.abs(d - x)) <= np.float32(5.0) / 255 * 0.5001


def test_qformat_closed_form_matches_two_peer_ring():
    rng = np.random.default_rng(2)
    bufs = [rng.normal(0, 1, 101).astype(np.float32) for _ in range(2)]
    out = oq.ring_allreduce_chunkwise_ex(bufs, oring.ReduceOp.SUM, "u16")
    # chunk 0 folds x0 then x1 (the owner is position 1), chunk 1 folds x1 then x0
    lo, hi = oring.chunk_bounds(101, 2)[0]
    a = oq.roundtrip(bufs[0][lo:hi], "u16")
    want = oq.roundtrip(bufs[1][lo:hi] + a, "u16")
    assert out[lo:hi].tobytes() == want.astype(np.float32).tobytes()
