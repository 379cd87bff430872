"""One-process-per-GPU ring all-reduce over NVLink (csrc/ring_ipc.cu).

``DeviceRing`` is the engine seam of the reference's ``run_all_reduce``
(collective.py:489-576): it runs one attempt of a tagged all-reduce over the
committed ring order on a CUDA tensor, in place, and raises
``CollectiveAborted`` after restoring the caller's bytes when the attempt is
aborted (host abort word, peer abort, timeout, injected fault, non-finite
quantized span).

torch.distributed is used only as plumbing: once per workspace it exchanges
the 64-byte CUDA IPC handles. The data path never calls NCCL.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native
from ._native import Stats, check, lib
from .collective import DTYPE_CODE, CollectiveAborted, ReduceOp, UsageError

_STATUS_REASON = {
    _native.PCCLB_EABORTED: ("abort signaled", "master"),
    _native.PCCLB_ETIMEOUT: ("io failure: peer timeout", "io"),
    _native.PCCLB_EIO: ("io failure: injected fault", "io"),
    _native.PCCLB_ENONFINITE: ("non-finite values cannot be quantized", "io"),
}


@dataclass
class ReduceStats:
    tx_payload_bytes: int
    rx_payload_bytes: int
    phase_ms: tuple = ()  # filled when PCCLB_RING_PROFILE=1 (csrc/ring_ipc.cu PhaseTimer)


class RingTicket:
    """An enqueued all-reduce attempt (the AsyncHandle of client.py:102-127)."""

    def __init__(self, ring: "DeviceRing", index: int, buffer: torch.Tensor, attempt: int = 0):
        self.ring = ring
        self.index = index
        self.buffer = buffer  # kept alive while the engine owns it
        self.attempt = attempt
        self.consumed = False


def exchange_bytes(payload: bytes, group=None) -> list[bytes]:
    """all_gather of a small byte string over the process group."""
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, payload, group=group)
    return out


class DeviceRing:
    """Ring engine for this process's GPU.

    ``ring`` lists global ranks in ring order (the master's committed ring,
    client.py:902); this rank's ring position is its index in it.
    """

    def __init__(self, group=None, ring: list[int] | None = None, device=None,
                 capacity_bytes: int = 64 << 20, timeout_s: float = 60.0, slots: int = 2,
                 small_max_bytes: int | None = None):
        if not dist.is_initialized():
            raise UsageError("torch.distributed must be initialized")
        self.group = group
        world = dist.get_world_size(group)
        me = dist.get_rank(group)
        self.ring = list(ring) if ring is not None else list(range(world))
        if sorted(self.ring) != list(range(world)):
            raise UsageError("ring must be a permutation of the group's ranks")
        self.position = self.ring.index(me)
        self.world = world
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.timeout_s = timeout_s
        self._attempt = 0
        self._handle = None
        self._capacity = 0
        self._registered: dict[int, torch.Tensor] = {}  # slot -> tensor (kept alive)
        self._pending = 0  # enqueued attempts not yet awaited
        # engines sharing this GPU concurrently (the communicator's pool size)
        self.slots = max(1, int(slots))
        # plain ops up to this size run as one fused kernel (None: library default, 4 MiB)
        self.small_max_bytes = small_max_bytes
        self._create(capacity_bytes)

    # -- workspace lifecycle (collective: every rank calls in the same order) --
    def _create(self, capacity_bytes: int) -> None:
        self._destroy()
        h = ctypes.c_void_p()
        check(
            lib().pcclb_ring_create(self.device.index, self.position, self.world, capacity_bytes, ctypes.byref(h)),
            "ring_create",
        )
        self._handle = h
        self._capacity = capacity_bytes
        check(lib().pcclb_ring_set_slots(h, self.slots), "ring_set_slots")
        if self.small_max_bytes is not None:
            check(lib().pcclb_ring_set_small_max(h, int(self.small_max_bytes)), "ring_set_small_max")
        mine = ctypes.create_string_buffer(64)
        check(lib().pcclb_ring_export(h, mine), "ring_export")
        handles = exchange_bytes(bytes(mine.raw), self.group)  # indexed by group rank
        for pos, grank in enumerate(self.ring):
            if pos == self.position:
                continue
            buf = ctypes.create_string_buffer(handles[grank], 64)
            check(lib().pcclb_ring_import(h, pos, buf), f"ring_import(peer {pos})")
        self._abort = lib().pcclb_ring_abort_word(h)
        for slot, t in sorted(self._registered.items()):
            self._register_slot(slot, t)

    def _destroy(self) -> None:
        if self._handle is not None:
            lib().pcclb_ring_destroy(self._handle)
            self._handle = None

    def close(self) -> None:
        self._destroy()

    def __del__(self):
        try:
            self._destroy()
        except Exception:
            pass

    @staticmethod
    def required_bytes(n: int, world: int, esz: int, quantize: bool) -> int:
        """Workspace bytes for an n-element op: the engine's own layout
        (pcclb_ring_workspace_bytes, host-only)."""
        code = 2 if esz == 8 else 1  # wire.py dtype codes: 1 f32, 2 f64
        need = int(lib().pcclb_ring_workspace_bytes(n, world, code, int(quantize)))
        if need == 0:
            raise UsageError(f"no workspace layout for n={n}, world={world}")
        return need + 4096

    def ensure_capacity(self, n: int, dtype: torch.dtype, quantize: bool) -> None:
        """Grow the workspace for an n-element op. Growing is collective (every
        rank re-exports its workspace), so it is refused while attempts are in
        flight, and the ranks first agree on (n, dtype, quantize): SPMD callers
        all reach this point together; ranks that disagree all raise
        UsageError. (A rank whose op still fits does not take part -- with
        mismatched sizes that rank's attempt then fails at its first barrier.)"""
        code = DTYPE_CODE[dtype]
        if lib().pcclb_ring_capacity(self._handle, code, int(quantize)) >= n:
            return
        if self._pending:
            raise UsageError("workspace must grow, but attempts are in flight: await them first")
        key = (int(n), int(code), bool(quantize))
        keys: list = [None] * self.world
        dist.all_gather_object(keys, key, group=self.group)
        if any(k != key for k in keys):
            raise UsageError(f"ranks disagree on the op that grows the workspace: {sorted(set(keys))}")
        esz = torch.tensor([], dtype=dtype).element_size()
        self._create(self.required_bytes(n, self.world, esz, quantize))

    def set_small_max_bytes(self, nbytes: int | None) -> None:
        """Largest op (bytes) that takes the one-kernel small path; None = the
        engine default. Every rank must set the same value (the path is part
        of the op descriptor the barrier compares)."""
        self.small_max_bytes = nbytes
        if self._handle:
            check(lib().pcclb_ring_set_small_max(self._handle, (1 << 64) - 1 if nbytes is None else int(nbytes)),
                  "ring_set_small_max")

    # -- caller-buffer registration (collective, SPMD order) --
    def register(self, tensor: torch.Tensor) -> int:
        """Register a CUDA tensor on every rank (all ranks call with their
        counterpart tensor, in the same order). All-reduces on (slices of) it
        then read it in place over NVLink. Returns the registration slot; the
        engine keeps the tensor alive until ``deregister``."""
        if not isinstance(tensor, torch.Tensor) or not tensor.is_cuda or not tensor.is_contiguous():
            raise UsageError("register needs a contiguous CUDA tensor")
        slot = 0
        while slot in self._registered:
            slot += 1
        self._register_slot(slot, tensor)
        self._registered[slot] = tensor
        return slot

    def _register_slot(self, slot: int, tensor: torch.Tensor) -> None:
        handle = ctypes.create_string_buffer(64)
        off = ctypes.c_uint64()
        check(lib().pcclb_ipc_handle(tensor.data_ptr(), handle, ctypes.byref(off)), "ipc_handle")
        allv = exchange_bytes(bytes(handle.raw) + int(off.value).to_bytes(8, "little"), self.group)
        handles = b"".join(allv[g][:64] for g in self.ring)
        offsets = (ctypes.c_uint64 * self.world)(*[int.from_bytes(allv[g][64:72], "little") for g in self.ring])
        hbuf = ctypes.create_string_buffer(handles, len(handles))
        nbytes = tensor.numel() * tensor.element_size()
        check(lib().pcclb_ring_register(self._handle, slot, tensor.data_ptr(), nbytes, hbuf, offsets), "ring_register")

    def deregister(self, slot: int) -> None:
        if slot in self._registered:
            check(lib().pcclb_ring_deregister(self._handle, slot), "ring_deregister")
            del self._registered[slot]

    # -- control-plane hooks --
    def signal_abort(self, attempt: int | None = None) -> None:
        """Abort attempts up to `attempt` (the tag box abort_event set on
        ABORT_NOTIFY, client.py:196-204). The word is attempt-scoped: it
        aborts every attempt <= the value at its next barrier, vote or poll,
        and no later one. Default: the attempt in flight and the next one
        enqueued (an abort raised just before the op)."""
        a = self._attempt + 1 if attempt is None else int(attempt)
        if a > self._abort[0]:
            self._abort[0] = a

    def reset_abort(self) -> None:
        """Kept for the reference's box.reset_for_attempt call sites: an
        attempt-scoped abort word never needs clearing."""

    # -- the op --
    def _validate(self, buffer: torch.Tensor, op, quantize: bool):
        op = ReduceOp.parse(op)
        if not isinstance(buffer, torch.Tensor) or buffer.dim() != 1 or not buffer.is_contiguous():
            raise UsageError("buffer must be a one-dimensional contiguous tensor")
        if buffer.device != self.device:
            raise UsageError(f"buffer must live on {self.device}")
        if buffer.dtype not in DTYPE_CODE:
            raise UsageError(f"unsupported dtype {buffer.dtype}")
        if quantize and buffer.dtype != torch.float32:
            raise UsageError("quantization requires float32 buffers")
        if quantize not in (False, True, None, "u8"):
            raise UsageError(f"the NVLink engine quantizes u8 min-max only (the reference's format), not {quantize!r}")
        return op

    def all_reduce_async(self, buffer: torch.Tensor, op=ReduceOp.SUM, quantize: bool = False,
                         fault_at: int = -1, stream: torch.cuda.Stream | None = None) -> "RingTicket":
        """Enqueue one attempt on `stream` and return at once (the engine owns
        the buffer until the ticket is awaited; client.py:802-827)."""
        op = self._validate(buffer, op, quantize)
        n = buffer.numel()
        self.ensure_capacity(n, buffer.dtype, quantize)
        self._attempt += 1
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        t = ctypes.c_uint32()
        rc = lib().pcclb_ring_enqueue(
            self._handle, buffer.data_ptr(), n, DTYPE_CODE[buffer.dtype], op.code, int(quantize),
            self._attempt, fault_at, self.timeout_s, s, ctypes.byref(t),
        )
        self._raise_for(rc, "ring_enqueue")
        self._pending += 1
        return RingTicket(self, int(t.value), buffer, self._attempt)

    def _raise_for(self, rc: int, what: str) -> None:
        if rc == _native.PCCLB_OK:
            return
        if rc == _native.PCCLB_EINVAL:
            raise UsageError("ring all-reduce rejected its arguments (ranks must agree on size, dtype, "
                             "op, quantization and buffer registration)")
        if rc in _STATUS_REASON:
            reason, source = _STATUS_REASON[rc]
            raise CollectiveAborted(reason, source=source)
        check(rc, what)

    def await_reduce(self, ticket: "RingTicket") -> ReduceStats:
        """Block until the attempt resolves; raises CollectiveAborted after the
        buffer was restored (collective.py:568-574). Every rank reaches the
        same outcome: the attempt ends with a completion vote on the device
        (the reference's COLLECTIVE_COMPLETE_VOTE), and a failure anywhere
        restores the buffers of all ranks."""
        if ticket.consumed:
            raise UsageError("ticket already awaited")
        ticket.consumed = True
        self._pending -= 1
        stats = Stats()
        rc = lib().pcclb_ring_wait(self._handle, ticket.index, ctypes.byref(stats))
        self._raise_for(rc, "ring_wait")
        phases = tuple(round(stats.phase_ms[i], 4) for i in range(stats.n_phases))
        return ReduceStats(stats.tx_payload_bytes, stats.rx_payload_bytes, phases)

    def run_all_reduce(self, buffer: torch.Tensor, op=ReduceOp.SUM, quantize: bool = False,
                       fault_at: int = -1, stream: torch.cuda.Stream | None = None) -> ReduceStats:
        """Synchronous attempt: enqueue + await (run_all_reduce, collective.py:489)."""
        return self.await_reduce(self.all_reduce_async(buffer, op, quantize, fault_at, stream))

    def restore(self, buffer: torch.Tensor) -> None:
        """Hand back the last op's input bytes (completion veto, client.py:973-983)."""
        self._validate(buffer, ReduceOp.SUM, False)
        check(
            lib().pcclb_ring_restore(self._handle, buffer.data_ptr(), buffer.numel(), DTYPE_CODE[buffer.dtype],
                                     torch.cuda.current_stream(self.device).cuda_stream),
            "ring_restore",
        )


def init_from_env(backend: str | None = None) -> tuple[int, int, int]:
    """torchrun-style init (RANK / WORLD_SIZE / LOCAL_RANK / MASTER_*)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    if not dist.is_initialized():
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend or "gloo", rank=rank, world_size=world)
    return rank, world, local
