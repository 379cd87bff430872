"""The product entry points fail loudly instead of handing a kernel a pointer
it cannot use: host tensors, wrong dtypes, unknown ops and a missing native
library are errors raised before any launch (no CPU fallback exists).
Mirrors the reference's synchronous UsageError checks (client.py:812-824,
bindings test_bindings.py:64-80). Runs without a GPU."""

from __future__ import annotations

import types

import pytest
import torch

from paper_2505_14065_b200 import _native
from paper_2505_14065_b200.collective import (
    ReduceOp,
    UsageError,
    accumulate,
    dequant_accumulate,
    dequantize_into,
    finalize_reduction,
    qformat_code,
    quantize_chunk,
    quantize_chunk_async,
)
from paper_2505_14065_b200.outer import PlainSGD, pseudo_gradient
from paper_2505_14065_b200.sharedstate import crc32_many, simplehash_many, simplehash_many_async

F = torch.zeros(16, dtype=torch.float32)
U8 = torch.zeros(16, dtype=torch.uint8)


@pytest.mark.parametrize(
    "call",
    [
        lambda: accumulate("sum", F.clone(), F.clone()),
        lambda: finalize_reduction(F.clone(), "avg", 2),
        lambda: quantize_chunk(F.clone(), U8.clone()),
        lambda: quantize_chunk_async(F.clone(), U8.clone(),
                                     types.SimpleNamespace(range=torch.zeros(4, dtype=torch.int32),
                                                           meta=torch.zeros(2))),
        lambda: dequantize_into(U8.clone(), 0.0, 1.0, F.clone()),
        lambda: dequant_accumulate("sum", F.clone(), U8.clone(), torch.zeros(2)),
        lambda: simplehash_many_async([U8.clone()], torch.zeros(1, dtype=torch.int64)),
        lambda: simplehash_many([U8.clone()]),
        lambda: crc32_many([U8.clone()]),
        lambda: pseudo_gradient(F.clone(), F.clone()),
        lambda: PlainSGD().step(F.clone(), F.clone()),
    ],
)
def test_host_tensors_are_rejected_before_any_launch(call):
    with pytest.raises(UsageError):
        call()


def test_non_tensors_are_rejected():
    with pytest.raises(UsageError):
        accumulate("sum", [1.0, 2.0], [3.0, 4.0])
    with pytest.raises(UsageError):
        finalize_reduction(bytearray(8), "avg", 2)


def test_unknown_reduce_op():
    with pytest.raises(UsageError):
        ReduceOp.parse("median")
    assert ReduceOp.parse("AVG") is ReduceOp.AVG
    assert ReduceOp.parse(5) is ReduceOp.PROD


def test_unknown_quantization_format():
    assert qformat_code(False) == 0 and qformat_code(True) == 1 and qformat_code("u16_zp") == 4
    with pytest.raises(UsageError):
        qformat_code("fp8")


def test_missing_library_raises(monkeypatch):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", "/nonexistent/libpcclb200.so")
    with pytest.raises(_native.NativeLibraryMissing):
        _native.lib()


def test_communicator_needs_torch_distributed():
    import torch.distributed as dist

    from paper_2505_14065_b200.communicator import Communicator

    if dist.is_initialized():
        pytest.skip("a process group is already initialised in this process")
    with pytest.raises(UsageError):
        Communicator()
