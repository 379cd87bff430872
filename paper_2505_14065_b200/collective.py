"""Device-side mirror of the reference's collective kernel seams.

Same names, argument meaning and error behaviour as
``/root/reference/pkg/src/churncomm/collective.py``, but the buffers are CUDA
``torch.Tensor`` objects and the arithmetic runs in libpcclb200's sm_100a
kernels (bit-identical to the reference's NumPy results). Calls are issued on
``torch.cuda.current_stream()``.

    ReduceOp                 collective.py:43-64   (wire codes wire.py:141-145)
    compute_chunk_boundaries collective.py:86-101
    quantize_chunk           collective.py:109-129
    dequantize_into          collective.py:132-135
    finalize_reduction       collective.py:479-482
    accumulate               collective.py:66-71 (_ACCUMULATE[op](a, b, out=a))
    CollectiveAborted        collective.py:77-83
"""

from __future__ import annotations

import ctypes
from enum import Enum

import torch

from . import _native
from ._native import F32, F64, QMeta, Range, check, lib


class UsageError(Exception):
    """Synchronous misuse (reference client.py:81-82, bindings UsageError)."""


class CollectiveAborted(Exception):
    """The attempt was cancelled; the caller's buffer has been restored."""

    def __init__(self, reason: str, source: str = "io"):
        super().__init__(reason)
        self.reason = reason
        self.source = source  # "master" | "io"


class ReduceOp(Enum):
    SUM = "sum"
    AVG = "avg"
    MAX = "max"
    MIN = "min"
    # extension (north_star): np.multiply in the same fold order; not in the
    # reference's ReduceOpCode (wire.py:141-145), so off-box frames reject it
    PROD = "prod"

    @property
    def code(self) -> int:
        return _OP_CODE[self]

    @classmethod
    def from_code(cls, code: int) -> "ReduceOp":
        return _CODE_OP[int(code)]

    @classmethod
    def parse(cls, op) -> "ReduceOp":
        if isinstance(op, ReduceOp):
            return op
        if isinstance(op, str):
            try:
                return cls(op.lower())
            except ValueError:
                raise UsageError(f"unknown reduce op {op!r}") from None
        if hasattr(op, "value") and isinstance(op.value, str):  # churncomm.ReduceOp
            return cls(op.value)
        return cls.from_code(int(op))


_OP_CODE = {ReduceOp.SUM: 1, ReduceOp.AVG: 2, ReduceOp.MAX: 3, ReduceOp.MIN: 4, ReduceOp.PROD: 5}
_CODE_OP = {v: k for k, v in _OP_CODE.items()}

# quantization formats (pcclb200.h PCCLB_Q_*): "u8" is the reference's
# min-max u8 (collective.py:109-135); the others are extensions (parity
# unpinned, oracle/quant_ext.py) that the single-GPU paths accept
QFORMATS = {"u8": 1, "u16": 2, "u8_zp": 3, "u16_zp": 4}


def qformat_code(quantize) -> int:
    """0 for no quantization, else the PCCLB_Q_* code of `quantize` (a bool --
    True is the reference's u8 -- or a format name)."""
    if quantize is None or quantize is False:
        return 0
    if quantize is True:
        return QFORMATS["u8"]
    if isinstance(quantize, str) and quantize in QFORMATS:
        return QFORMATS[quantize]
    raise UsageError(f"unknown quantization format {quantize!r} (one of {sorted(QFORMATS)})")

# torch.bfloat16 (code 3) is an extension (pcclb200.h PCCLB_BF16): plain ops
# on the single-GPU and NVLink paths; the reference's wire has f32/f64 only
DTYPE_CODE = {torch.float32: F32, torch.float64: F64, torch.bfloat16: 3}


def compute_chunk_boundaries(n_elements: int, world_size: int) -> list[tuple[int, int]]:
    """Contiguous per-rank element ranges partitioning [0, n_elements)."""
    if world_size < 1:
        raise ValueError("world_size must be at least 1")
    out = (ctypes.c_uint64 * (2 * world_size))()
    check(lib().pcclb_chunk_bounds(n_elements, world_size, out), "chunk_bounds")
    return [(int(out[2 * r]), int(out[2 * r + 1])) for r in range(world_size)]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _check_buffer(t: torch.Tensor, what: str, dtypes=(torch.float32, torch.float64, torch.bfloat16),
                  min_numel: int = 0, device: torch.device | None = None) -> None:
    """Every pointer handed to a kernel is checked first: a host, undersized or
    other-device tensor is a UsageError here, never a device fault."""
    if not isinstance(t, torch.Tensor):
        raise UsageError(f"{what} must be a torch.Tensor")
    if not t.is_cuda:
        raise UsageError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise UsageError(f"{what} must be contiguous")
    if dtypes is not None and t.dtype not in dtypes:
        raise UsageError(f"{what} has unsupported dtype {t.dtype}")
    if t.numel() < min_numel:
        raise UsageError(f"{what} has {t.numel()} elements, needs {min_numel}")
    if device is not None and t.device != device:
        raise UsageError(f"{what} is on {t.device}, the operation runs on {device}")


def accumulate(op, acc: torch.Tensor, incoming: torch.Tensor) -> None:
    """``acc <- acc (+) incoming`` in place (np.add / np.maximum / np.minimum)."""
    op = ReduceOp.parse(op)
    _check_buffer(acc, "acc")
    _check_buffer(incoming, "incoming", device=acc.device)
    if acc.dtype != incoming.dtype or acc.numel() != incoming.numel():
        raise UsageError("acc and incoming must match in dtype and size")
    with torch.cuda.device(acc.device):
        check(
            lib().pcclb_accumulate(
                acc.data_ptr(), incoming.data_ptr(), acc.numel(), DTYPE_CODE[acc.dtype], op.code, _stream()
            ),
            "accumulate",
        )


def finalize_reduction(buffer: torch.Tensor, op, world_size: int) -> None:
    """Average divides by world size; other operators are complete as-is."""
    op = ReduceOp.parse(op)
    _check_buffer(buffer, "buffer")
    with torch.cuda.device(buffer.device):
        check(
            lib().pcclb_finalize(
                buffer.data_ptr(), buffer.numel(), DTYPE_CODE[buffer.dtype], op.code, world_size, _stream()
            ),
            "finalize_reduction",
        )


class QuantScratch:
    """Device range + meta slots for one quantized span (reused across calls)."""

    def __init__(self, device):
        self.range = torch.zeros(4, dtype=torch.int32, device=device)  # pcclb_range
        self.meta = torch.zeros(2, dtype=torch.float32, device=device)  # pcclb_qmeta


def quantize_chunk_async(values: torch.Tensor, out: torch.Tensor, scratch: QuantScratch,
                         adopt: torch.Tensor | None = None, avg_div: int = 1) -> None:
    """Device-only quantize: range, then codes; (min, scale) land in
    ``scratch.meta`` and the non-finite flag in ``scratch.range[2]``."""
    _check_buffer(values, "values", (torch.float32,))
    n = values.numel()
    dev = values.device
    _check_buffer(out, "out", (torch.uint8,), n, dev)
    _check_buffer(scratch.range, "scratch.range", (torch.int32,), 4, dev)
    _check_buffer(scratch.meta, "scratch.meta", (torch.float32,), 2, dev)
    if adopt is not None:
        _check_buffer(adopt, "adopt", (torch.float32,), n, dev)
    with torch.cuda.device(dev):
        s = _stream()
        L = lib()
        check(L.pcclb_range_reset(scratch.range.data_ptr(), 1, s), "range_reset")
        check(L.pcclb_range_f32(values.data_ptr(), n, scratch.range.data_ptr(), s), "range_f32")
        check(
            L.pcclb_quantize_u8(
                values.data_ptr(),
                n,
                scratch.range.data_ptr(),
                out.data_ptr(),
                scratch.meta.data_ptr(),
                adopt.data_ptr() if adopt is not None else None,
                avg_div,
                s,
            ),
            "quantize_u8",
        )


def quantize_chunk(values: torch.Tensor, out: torch.Tensor) -> tuple[float, float]:
    """Quantize a float32 span into u8 codes; returns (min_val, scale).

    q = round((x - min) / scale) clamped to [0, 255] with
    scale = (max - min) / 255, or 1 when the span is constant. Raises
    ValueError on non-finite input, like the reference (collective.py:117-118).
    """
    _check_buffer(values, "values", (torch.float32,))
    _check_buffer(out, "out", (torch.uint8,), values.numel(), values.device)
    if values.numel() == 0:
        return 0.0, 1.0
    scratch = QuantScratch(values.device)
    quantize_chunk_async(values, out, scratch)
    flags = scratch.range.cpu()
    if int(flags[2]) != 0:
        raise ValueError("non-finite values cannot be quantized")
    meta = scratch.meta.cpu()
    return float(meta[0]), float(meta[1])


def _meta_tensor(min_val: float, scale: float, device) -> torch.Tensor:
    return torch.tensor([min_val, scale], dtype=torch.float32).to(device, non_blocking=False)


def dequantize_into(codes: torch.Tensor, min_val: float, scale: float, out: torch.Tensor) -> None:
    """Inverse mapping x = min + q * scale, written into out (float32)."""
    _check_buffer(out, "out", (torch.float32,))
    n = out.numel()
    _check_buffer(codes, "codes", (torch.uint8,), n, out.device)
    meta = _meta_tensor(min_val, scale, out.device)
    with torch.cuda.device(out.device):
        check(
            lib().pcclb_dequantize_u8(out.data_ptr(), codes.data_ptr(), n, meta.data_ptr(), 1, _stream()),
            "dequantize_u8",
        )


def dequant_accumulate(op, acc: torch.Tensor, codes: torch.Tensor, meta: torch.Tensor,
                       next_range: torch.Tensor | None = None) -> None:
    """Quantized reduce consume (collective.py:399-409): acc <- acc (+) D(codes)."""
    op = ReduceOp.parse(op)
    _check_buffer(acc, "acc", (torch.float32,))
    n, dev = acc.numel(), acc.device
    _check_buffer(codes, "codes", (torch.uint8,), n, dev)
    _check_buffer(meta, "meta", (torch.float32,), 2, dev)
    if next_range is not None:
        _check_buffer(next_range, "next_range", (torch.int32,), 4, dev)
    with torch.cuda.device(dev):
        check(
            lib().pcclb_dequant_accumulate_u8(
                acc.data_ptr(),
                codes.data_ptr(),
                n,
                meta.data_ptr(),
                op.code,
                next_range.data_ptr() if next_range is not None else None,
                _stream(),
            ),
            "dequant_accumulate_u8",
        )


__all__ = [
    "ReduceOp",
    "UsageError",
    "CollectiveAborted",
    "compute_chunk_boundaries",
    "accumulate",
    "finalize_reduction",
    "quantize_chunk",
    "quantize_chunk_async",
    "dequantize_into",
    "dequant_accumulate",
    "QuantScratch",
    "Range",
    "QMeta",
    "_native",
]
