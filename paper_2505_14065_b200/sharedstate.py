"""Device-side mirror of the reference's shared-state hashing.

Mirrors ``/root/reference/pkg/src/churncomm/sharedstate.py``:

    simplehash(buffer, workers=1) -> int     sharedstate.py:87-105
    SharedStateEntry / content_hash          sharedstate.py:136-172
    digest_entries(entries)                  sharedstate.py:175-178

``buffer`` is a CUDA tensor (hashed in place over its raw bytes) or any host
buffer (bytes / NumPy / CPU tensor), which is streamed host->device through
pinned staging and hashed with the resumable kernel. ``workers`` is accepted
for signature compatibility; the result is independent of it, as in the
reference. ``digest_entries`` hashes all entries in ONE multi-entry launch.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import IntEnum

import torch

from ._native import check, lib
from .collective import UsageError

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
LANES = 256
TREE_DEPTH = 8
ROTATE = 27


class DType(IntEnum):
    """wire.py:130-138"""

    F32 = 1
    F64 = 2
    U8 = 3
    I32 = 4
    I64 = 5


DTYPE_WIDTH = {DType.F32: 4, DType.F64: 8, DType.U8: 1, DType.I32: 4, DType.I64: 8}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _device_bytes(t: torch.Tensor, device: torch.device) -> tuple[int, int]:
    # checked before any launch: a host or other-device pointer must be a
    # UsageError, not a device fault
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise UsageError("hashed buffers must be CUDA tensors")
    if t.device != device:
        raise UsageError(f"hashed buffers must all live on {device} (got {t.device})")
    if not t.is_contiguous():
        raise ValueError("buffer must be contiguous")
    return t.data_ptr(), t.numel() * t.element_size()


def _check_out(out: torch.Tensor, dtype: torch.dtype, n: int) -> None:
    if not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != dtype or not out.is_contiguous():
        raise UsageError(f"out must be a contiguous CUDA {dtype} tensor")
    if out.numel() < n:
        raise UsageError(f"out has {out.numel()} slots for {n} digests")


def _to_u64(v: torch.Tensor) -> list[int]:
    return [int(x) & 0xFFFFFFFFFFFFFFFF for x in v.cpu().tolist()]


def simplehash_many_async(tensors: list[torch.Tensor], out: torch.Tensor) -> None:
    """Hash CUDA tensors into ``out`` (int64 CUDA tensor, bit pattern = u64)."""
    n = len(tensors)
    if n == 0:
        return
    _check_out(out, torch.int64, n)
    ptrs = (ctypes.c_void_p * n)()
    sizes = (ctypes.c_uint64 * n)()
    for i, t in enumerate(tensors):
        p, nb = _device_bytes(t, out.device)
        ptrs[i] = p
        sizes[i] = nb
    with torch.cuda.device(out.device):
        check(lib().pcclb_simplehash_multi(ptrs, sizes, n, out.data_ptr(), _stream()), "simplehash_multi")


def simplehash_many(tensors: list[torch.Tensor]) -> list[int]:
    if not tensors:
        return []
    if not isinstance(tensors[0], torch.Tensor) or not tensors[0].is_cuda:
        raise UsageError("hashed buffers must be CUDA tensors")
    dev = tensors[0].device
    out = torch.empty(len(tensors), dtype=torch.int64, device=dev)
    simplehash_many_async(tensors, out)
    return _to_u64(out)


def crc32_many(tensors: list[torch.Tensor]) -> list[int]:
    """zlib.crc32 of the raw bytes of CUDA tensors, one launch for all
    (extension digest, csrc/crc.cu; parity pinned by zlib)."""
    n = len(tensors)
    if n == 0:
        return []
    if not isinstance(tensors[0], torch.Tensor) or not tensors[0].is_cuda:
        raise UsageError("crc32 buffers must be CUDA tensors")
    dev = tensors[0].device
    ptrs = (ctypes.c_void_p * n)()
    sizes = (ctypes.c_uint64 * n)()
    for i, t in enumerate(tensors):
        p, nb = _device_bytes(t, dev)
        ptrs[i] = p
        sizes[i] = nb
    out = torch.empty(n, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        check(lib().pcclb_crc32_multi(ptrs, sizes, n, out.data_ptr(), _stream()), "crc32_multi")
    return [int(x) & 0xFFFFFFFF for x in out.cpu().tolist()]


def crc32(tensor: torch.Tensor) -> int:
    """zlib.crc32 of a CUDA tensor's bytes."""
    return crc32_many([tensor])[0]


class StreamingHasher:
    """Hash a host byte stream on the GPU: pinned double-buffered staging,
    H2D copy of segment i+1 overlapped with hashing of segment i."""

    def __init__(self, device=None, segment_bytes: int = 64 << 20):
        self.device = torch.device(device or "cuda")
        self.segment = max(1024, segment_bytes - segment_bytes % 1024)
        self.pinned = [torch.empty(self.segment, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.dev = [torch.empty(self.segment, dtype=torch.uint8, device=self.device) for _ in range(2)]
        self.state = torch.empty(LANES, dtype=torch.int64, device=self.device)
        self.out = torch.empty(1, dtype=torch.int64, device=self.device)
        self.copy_stream = torch.cuda.Stream(self.device)
        self.events = [torch.cuda.Event() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]

    def hash(self, data) -> int:
        if isinstance(data, torch.Tensor):
            mv = data.contiguous().view(torch.uint8).reshape(-1)
            src = mv if mv.device.type == "cpu" else mv.cpu()
        else:
            src = torch.frombuffer(bytearray(memoryview(data).cast("B")), dtype=torch.uint8) if len(memoryview(data).cast("B")) else torch.empty(0, dtype=torch.uint8)
        total = src.numel()
        L = lib()
        s = torch.cuda.current_stream(self.device)
        check(L.pcclb_simplehash_init(self.state.data_ptr(), s.cuda_stream), "simplehash_init")
        off, k = 0, 0
        while off < total:
            nb = min(self.segment, total - off)
            b = k % 2
            # staging slot b is free once the hash that read it (2 segments ago) finished
            self.done[b].synchronize()
            self.pinned[b][:nb].copy_(src[off : off + nb])
            with torch.cuda.stream(self.copy_stream):
                self.copy_stream.wait_event(self.done[b])
                self.dev[b][:nb].copy_(self.pinned[b][:nb], non_blocking=True)
                self.events[b].record(self.copy_stream)
            s.wait_event(self.events[b])
            check(L.pcclb_simplehash_update(self.state.data_ptr(), self.dev[b].data_ptr(), nb, s.cuda_stream), "simplehash_update")
            self.done[b].record(s)
            off += nb
            k += 1
        check(L.pcclb_simplehash_final(self.state.data_ptr(), total, self.out.data_ptr(), s.cuda_stream), "simplehash_final")
        return _to_u64(self.out)[0]


_hasher: StreamingHasher | None = None


def simplehash(buffer, workers: int = 1) -> int:
    """64-bit content hash, identical to the reference for any worker count."""
    if isinstance(buffer, torch.Tensor) and buffer.is_cuda:
        return simplehash_many([buffer])[0]
    global _hasher
    if _hasher is None:
        _hasher = StreamingHasher()
    return _hasher.hash(buffer)


@dataclass
class SharedStateEntry:
    """One keyed, caller-owned buffer participating in state sync
    (sharedstate.py:136-172). Hashing covers the raw bytes."""

    key: str
    dtype: DType
    buffer: torch.Tensor
    revision: int = 0

    def __post_init__(self):
        width = DTYPE_WIDTH[DType(self.dtype)]
        if self.nbytes % width:
            raise ValueError(f"entry {self.key!r}: {self.nbytes} bytes not divisible by element width {width}")

    @property
    def nbytes(self) -> int:
        return self.buffer.numel() * self.buffer.element_size()

    def content_hash(self, workers: int = 1) -> int:
        return simplehash(self.buffer, workers=workers)


def digest_entries(entries: list[SharedStateEntry]) -> list[tuple[str, int, int]]:
    """Per-entry (key, revision, hash) triples from one multi-entry launch."""
    hashes = simplehash_many([e.buffer for e in entries])
    return [(e.key, e.revision, h) for e, h in zip(entries, hashes)]
