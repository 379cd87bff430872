"""Ring all-reduce engines.

``LocalRing`` -- W logical peers whose buffers live on one GPU: the
B200-side counterpart of the reference's in-process ``RingSession``
(tests/ring_harness.py:24-105), used for single-GPU parity runs and the
single-GPU benchmark. The schedule is the reference's (collective.py:489-567);
see csrc/ring_local.cu for how it maps onto kernels.

``DeviceRing`` (ring_ipc.py) is the one-process-per-GPU NVLink engine.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native
from ._native import check, lib
from .collective import DTYPE_CODE, CollectiveAborted, ReduceOp, UsageError, qformat_code


class LocalRing:
    """A fixed ring of W logical peers on one CUDA device."""

    def __init__(self, world: int, device=None, backup: bool = True):
        if world < 1 or world > 64:
            raise UsageError("world must be in [1, 64]")
        self.world = world
        dev = torch.device(device or "cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.backup_enabled = backup
        nbytes = int(lib().pcclb_local_scratch_bytes(world))
        self.scratch = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=self.device)
        self._backup: torch.Tensor | None = None

    def _backup_buf(self, n: int, dtype) -> torch.Tensor:
        need = self.world * n
        if self._backup is None or self._backup.numel() < need or self._backup.dtype != dtype:
            self._backup = torch.empty(need, dtype=dtype, device=self.device)  # pool: reused
        return self._backup

    def launch(self, buffers: list[torch.Tensor], op, quantize=False, stream=None) -> int:
        """Enqueue the op on `stream` (plain ops never block the host);
        returns the raw status. `quantize`: False, True (the reference's u8
        min-max) or an extension format name ("u16", "u8_zp", "u16_zp")."""
        op = ReduceOp.parse(op)
        qf = qformat_code(quantize)
        if len(buffers) != self.world:
            raise UsageError(f"expected {self.world} buffers")
        b0 = buffers[0]
        for b in buffers:
            if not isinstance(b, torch.Tensor) or not b.is_cuda or b.dim() != 1 or not b.is_contiguous():
                raise UsageError("buffers must be 1-D contiguous CUDA tensors")
            if b.dtype != b0.dtype or b.numel() != b0.numel() or b.device != self.device:
                raise UsageError("buffers must agree in dtype, size and device")
        if b0.dtype not in DTYPE_CODE:
            raise UsageError(f"unsupported dtype {b0.dtype}")
        if quantize and b0.dtype != torch.float32:
            raise UsageError("quantization requires float32 buffers")
        n = b0.numel()
        ptrs = (ctypes.c_void_p * self.world)(*[b.data_ptr() for b in buffers])
        backup = self._backup_buf(n, b0.dtype).data_ptr() if (self.backup_enabled and quantize) else None
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        return lib().pcclb_local_allreduce_ex(
            ptrs, self.world, n, DTYPE_CODE[b0.dtype], op.code, qf, self.scratch.data_ptr(), backup, s
        )

    def run_op(self, buffers: list[torch.Tensor], op, quantize=False) -> list[tuple[str, object]]:
        """Run one attempt on all ranks; per-rank (status, extra) like RingSession.run_op."""
        rc = self.launch(buffers, op, quantize)
        if rc == _native.PCCLB_OK:
            return [("ok", None)] * self.world
        if rc == _native.PCCLB_ENONFINITE:
            err = CollectiveAborted("non-finite values cannot be quantized", source="io")
            return [("aborted", err)] * self.world
        check(rc, "local_allreduce")
        raise AssertionError("unreachable")
