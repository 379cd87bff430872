"""North-star extensions absent from the reference (SURVEY §0, §8c "parity
unpinned"): their oracle is this repo's own restatement in oracle/, defined
the way the reference defines its ops (same fold order, same rounding rules),
and the GPU paths must match it bit for bit.

  PROD   np.multiply folded in the ring order (oracle/ring.py ReduceOp.PROD)
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ring as oring
from tests.gpu_util import bits, need_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _prod_inputs(w: int, n: int, dtype, seed: int) -> list[np.ndarray]:
    # factors near 1 keep W-fold products finite; a few exact edge values
    rng = np.random.default_rng(seed)
    out = []
    for p in range(w):
        x = (1.0 + 0.05 * rng.normal(0, 1, n)).astype(dtype)
        if n > 8:
            x[:4] = np.array([0.0, -0.0, 2.0, -1.5], dtype=dtype)[: 4]
        out.append(x)
    return out


@pytest.mark.parametrize("w", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("n", [0, 1, 7, 4099, 100_003])
@pytest.mark.parametrize("dtype,quant", [(np.float32, False), (np.float64, False), (np.float32, True)])
def test_prod_local_ring(w, n, dtype, quant):
    from paper_2505_14065_b200 import LocalRing

    host = _prod_inputs(w, n, dtype, 1000 * w + n)
    want = oring.ring_allreduce_chunkwise(host, oring.ReduceOp.PROD, quantize=quant)
    dev = [to_dev(h) for h in host]
    res = LocalRing(w).run_op(dev, "prod", quantize=quant)
    assert all(s == "ok" for s, _ in res)
    for d in dev:
        assert bits(d) == bits(want)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_prod_accumulate_kernel(dtype):
    from paper_2505_14065_b200.collective import accumulate

    rng = np.random.default_rng(5)
    npd = np.float32 if dtype == torch.float32 else np.float64
    a = rng.normal(0, 3, 100_001).astype(npd)
    b = rng.normal(0, 3, 100_001).astype(npd)
    a[:6] = [np.nan, 1.0, np.inf, 0.0, -0.0, 1e-40]
    b[:6] = [2.0, np.nan, 0.0, np.inf, 5.0, 1e-5]
    want = a.copy()
    oring.accumulate(oring.ReduceOp.PROD, want, b)
    da, db = to_dev(a), to_dev(b)
    accumulate("prod", da, db)
    assert bits(da) == bits(want)


# ---------------------------------------------------------------------------
# CRC-32 (csrc/crc.cu): the checker is zlib.crc32 itself
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [0, 1, 3, 15, 16, 17, 1023, 1024, 1025, 262143, 262144, 262145,
                               (1 << 20) + 7, (3 << 20) + 262144 * 2 + 5])
def test_crc32_sizes(n):
    import zlib

    from paper_2505_14065_b200 import crc32

    raw = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    assert crc32(to_dev(raw)) == zlib.crc32(raw.tobytes())


@pytest.mark.parametrize("offset", [1, 2, 5, 8, 13])
def test_crc32_misaligned(offset):
    import zlib

    from paper_2505_14065_b200 import crc32

    raw = np.random.default_rng(offset).integers(0, 256, (1 << 20) + 99, dtype=np.uint8)
    dev = to_dev(raw)
    assert crc32(dev[offset:]) == zlib.crc32(raw[offset:].tobytes())


def test_crc32_many_and_large():
    """A multi-entry call (config-4-like mix) and a 1.05 GB entry."""
    import zlib

    from paper_2505_14065_b200 import crc32_many

    rng = np.random.default_rng(3)
    sizes = [int(x) for x in rng.integers(0, 3 << 20, 40)] + [0, 1, 1050673152]
    host = [rng.integers(0, 256, s, dtype=np.uint8) for s in sizes]
    got = crc32_many([to_dev(h) for h in host])
    assert got == [zlib.crc32(h.tobytes()) for h in host]


# ---------------------------------------------------------------------------
# u16 and zero-point quantization (oracle/quant_ext.py)
# ---------------------------------------------------------------------------
FMTS = ["u16", "u8_zp", "u16_zp"]


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("w", [2, 3, 5, 8])
@pytest.mark.parametrize("n", [1, 7, 4099, 100_003])
@pytest.mark.parametrize("op", ["sum", "avg", "max", "prod"])
def test_qformat_local_ring(fmt, w, n, op):
    from oracle import quant_ext as oq
    from paper_2505_14065_b200 import LocalRing

    rng = np.random.default_rng(w * 100_000 + n)
    if op == "prod":
        host = [(1.0 + 0.05 * rng.normal(0, 1, n)).astype(np.float32) for _ in range(w)]
    else:
        host = [rng.normal(0.3 if fmt.endswith("zp") else 0, 1, n).astype(np.float32) for _ in range(w)]
    want = oq.ring_allreduce_chunkwise_ex(host, oring.ReduceOp[op.upper()], fmt)
    dev = [to_dev(h) for h in host]
    res = LocalRing(w).run_op(dev, op, quantize=fmt)
    assert all(s == "ok" for s, _ in res)
    for d in dev:
        assert bits(d) == bits(want)


@pytest.mark.parametrize("fmt", FMTS)
def test_qformat_kernel_seams(fmt):
    """quantize_ex / dequantize_ex / dequant_accumulate_ex codes and values."""
    import ctypes

    from oracle import quant_ext as oq
    from paper_2505_14065_b200 import _native
    from paper_2505_14065_b200.collective import QFORMATS

    L = _native.lib()
    qf = QFORMATS[fmt]
    rng = np.random.default_rng(11)
    x = rng.normal(0.5, 2, 300_007).astype(np.float32)
    x[:5] = [0.0, -0.0, 1e-30, -3.5, 7.25]
    codes_want, p0, scale = oq.quantize_ex(x, fmt)
    dx = to_dev(x)
    rng_buf = torch.zeros(16, dtype=torch.uint8, device="cuda")
    meta = torch.zeros(2, dtype=torch.float32, device="cuda")
    codes = torch.zeros(x.size, dtype=torch.int16 if "16" in fmt else torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert L.pcclb_range_reset(rng_buf.data_ptr(), 1, s) == 0
    assert L.pcclb_range_f32(dx.data_ptr(), x.size, rng_buf.data_ptr(), s) == 0
    assert L.pcclb_quantize_ex(dx.data_ptr(), x.size, rng_buf.data_ptr(), codes.data_ptr(), meta.data_ptr(),
                               None, 1, qf, s) == 0
    got_codes = codes.cpu().numpy().view(codes_want.dtype)
    assert got_codes.tobytes() == codes_want.tobytes()
    assert meta.cpu().numpy().tobytes() == np.array([p0, scale], np.float32).tobytes()
    out = torch.empty_like(dx)
    assert L.pcclb_dequantize_ex(out.data_ptr(), codes.data_ptr(), x.size, meta.data_ptr(), 1, qf, s) == 0
    assert bits(out) == bits(oq.dequantize_ex(codes_want, p0, scale, fmt))
    acc = to_dev(x[::-1].copy())
    assert L.pcclb_dequant_accumulate_ex(acc.data_ptr(), codes.data_ptr(), x.size, meta.data_ptr(), 1, None,
                                         qf, s) == 0
    want = x[::-1].copy()
    oring.accumulate(oring.ReduceOp.SUM, want, oq.dequantize_ex(codes_want, p0, scale, fmt))
    assert bits(acc) == bits(want)
    del ctypes


def test_qformat_rejected_by_nvlink_and_tcp_engines():
    from paper_2505_14065_b200.collective import UsageError, qformat_code

    assert qformat_code(True) == 1 and qformat_code(False) == 0 and qformat_code("u16_zp") == 4
    with pytest.raises(UsageError):
        qformat_code("fp8")
    del UsageError


# ---------------------------------------------------------------------------
# bf16 buffers (oracle/bf16.py): f32 arithmetic per fold step, RNE to bf16
# ---------------------------------------------------------------------------
def _bf16_inputs(w, n, seed, op):
    from oracle import bf16 as ob

    rng = np.random.default_rng(seed)
    if op == "prod":
        fl = [(1.0 + 0.05 * rng.normal(0, 1, n)).astype(np.float32) for _ in range(w)]
    else:
        fl = [rng.normal(0, 1, n).astype(np.float32) for _ in range(w)]
    out = [ob.from_f32(f) for f in fl]
    if n > 8:
        out[0][:3] = [0x0000, 0x8000, 0x7F80]  # +0, -0, +inf
    return out


@pytest.mark.parametrize("w", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("n", [1, 7, 4099, 100_003])
@pytest.mark.parametrize("op", ["sum", "avg", "max", "min", "prod"])
def test_bf16_local_ring(w, n, op):
    from oracle import bf16 as ob
    from paper_2505_14065_b200 import LocalRing

    host = _bf16_inputs(w, n, 7 * n + w, op)
    want = ob.ring_allreduce_chunkwise(host, oring.ReduceOp[op.upper()]) if w > 1 else (
        ob.from_f32(ob.to_f32(host[0]) / np.float32(1)) if op == "avg" else host[0])
    dev = [torch.from_numpy(h.view(np.int16).copy()).cuda().view(torch.bfloat16) for h in host]
    res = LocalRing(w).run_op(dev, op)
    assert all(s == "ok" for s, _ in res)
    for d in dev:
        assert d.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == want.tobytes()


@pytest.mark.parametrize("op", ["sum", "max", "prod"])
def test_bf16_accumulate_and_finalize(op):
    from oracle import bf16 as ob
    from paper_2505_14065_b200.collective import accumulate, finalize_reduction

    a, b = _bf16_inputs(2, 100_001, 3, op)
    da = torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    db = torch.from_numpy(b.view(np.int16).copy()).cuda().view(torch.bfloat16)
    accumulate(op, da, db)
    want = ob.accumulate(oring.ReduceOp[op.upper()], a, b)
    assert da.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == want.tobytes()
    finalize_reduction(da, "avg", 3)
    want = ob.from_f32(ob.to_f32(want) / np.float32(3))
    assert da.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == want.tobytes()
