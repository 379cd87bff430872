"""Communicator facade: the reference's collective API on the B200 data plane.

Mirrors the data-plane half of ``churncomm.client.Communicator``
(client.py:421-1033) for peers that share one box:

    all_reduce_async(buffer, tag, op, quantize) -> AsyncHandle   client.py:802-827
    await_async_reduce(handle, timeout) -> ReduceResult          client.py:829-843
    all_reduce(...)                                              client.py:845-847
    sync_shared_state(entries, strategy) -> SyncOutcomeResult    client.py:692-741
    get_world_size()                                             client.py:560-563

Tags map to pool slots (``tag % pool_size``, client.py:826); every slot owns
one NVLink engine (``DeviceRing``) and one CUDA stream, so ops of different
slots run concurrently and ops of one slot run in FIFO order, like the
reference's per-slot worker queue. The control plane (master, votes,
membership) is not rebuilt: ``torch.distributed`` carries the few host
exchanges (IPC handles, shared-state digests), parameter agreement is checked
on the device at the first barrier, and ``abort(tag)`` is the hook a master
link would call on ABORT_NOTIFY. A lost peer surfaces as a timeout abort;
survivors then build a new Communicator over their group (a new ring) and
retry, as the reference's apps do (algos.py:117-125).
"""

from __future__ import annotations

import ctypes
from collections import Counter
from dataclasses import dataclass, field
from enum import Enum

import torch
import torch.distributed as dist

from ._native import check, lib
from .collective import CollectiveAborted, ReduceOp, UsageError
from .ring_ipc import DeviceRing, RingTicket
from .sharedstate import SharedStateEntry, simplehash_many


class SyncStrategy(Enum):
    """wire.py SyncStrategy names (bound.py:38-42 strings)."""

    ENFORCE_POPULAR = "enforcePopular"
    SEND_ONLY = "sendOnly"
    RECEIVE_ONLY = "receiveOnly"


class SyncStatus(Enum):
    IN_SYNC = "in_sync"
    UPDATED = "updated"
    ERROR = "error"


@dataclass
class SyncOutcomeResult:
    """sharedstate.py:187-195"""

    status: SyncStatus
    updated_keys: list[str] = field(default_factory=list)
    reason: str = ""

    @property
    def ok(self) -> bool:
        return self.status is not SyncStatus.ERROR


@dataclass
class ReduceResult:
    """client.py:118-127"""

    status: str  # "completed" | "aborted"
    reason: str = ""
    tx_bytes: int = 0
    rx_bytes: int = 0

    @property
    def completed(self) -> bool:
        return self.status == "completed"


class AsyncHandle:
    """client.py:130-170: one tagged operation; awaited exactly once."""

    def __init__(self, tag: int, slot: int, ticket: RingTicket | None, early: ReduceResult | None = None):
        self.tag = tag
        self.slot = slot
        self.ticket = ticket
        self._early = early
        self._consumed = False

    @property
    def pending(self) -> bool:
        return not self._consumed


def select_sync_plan(reports: dict[int, tuple[SyncStrategy, list[tuple[str, int, int, int]]]]):
    """Donor and receivers per entry, restating master.select_sync_plan
    (master.py:909-976) without a committed floor: send-only peers are the
    only donors if any exist, receive-only peers never donate, the highest
    revision wins, then the most popular hash (ties: smallest hash, then
    smallest peer). reports[peer] = (strategy, [(key, revision, hash, nbytes, dtype)]).
    Returns {peer: [(key, donor, revision, hash)]} or an error string."""
    send_only = {p for p, (s, _) in reports.items() if s is SyncStrategy.SEND_ONLY}
    recv_only = {p for p, (s, _) in reports.items() if s is SyncStrategy.RECEIVE_ONLY}
    plan: dict[int, list] = {p: [] for p in reports}
    first = next(iter(reports.values()))[1]
    for idx, (key, *_rest) in enumerate(first):
        state = {p: r[1][idx] for p, r in reports.items()}
        candidates = set(send_only) if send_only else set(reports) - recv_only
        if not candidates:
            return f"no eligible donor for {key!r}: every peer is receive-only"
        max_rev = max(state[p][1] for p in candidates)
        current = [p for p in candidates if state[p][1] == max_rev]
        tally = Counter(state[p][2] for p in current)
        top = max(tally.values())
        winning = min(h for h, c in tally.items() if c == top)
        donor = min(p for p in current if state[p][2] == winning)
        for p, meta in state.items():
            if p != donor and (meta[1], meta[2]) != (state[donor][1], state[donor][2]):
                plan[p].append((key, donor, state[donor][1], state[donor][2]))
    return plan


class Communicator:
    def __init__(self, group=None, device=None, pool_size: int = 2, ring: list[int] | None = None,
                 timeout_s: float = 60.0, capacity_bytes: int = 64 << 20):
        if not dist.is_initialized():
            raise UsageError("torch.distributed must be initialized")
        if pool_size < 1:
            raise UsageError("pool_size must be >= 1")
        self.group = group
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.pool_size = pool_size
        self.engines = [DeviceRing(group, ring, self.device, capacity_bytes, timeout_s, slots=pool_size)
                        for _ in range(pool_size)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(pool_size)]
        self._handles: dict[int, AsyncHandle] = {}
        self.stats = {"reduce_attempts": 0, "reduce_completed": 0, "reduce_aborted": 0, "sync_calls": 0,
                      "sync_payload_rx": 0}

    # -- membership view ---------------------------------------------------
    def get_world_size(self) -> int:
        return self.engines[0].world

    @property
    def rank(self) -> int:
        return dist.get_rank(self.group)

    def close(self) -> None:
        for e in self.engines:
            e.close()

    def register(self, tensor: torch.Tensor) -> None:
        """Register a buffer with every slot's engine (zero-copy reads)."""
        for e in self.engines:
            e.register(tensor)

    # -- collectives (client.py:802-847) -----------------------------------
    def all_reduce_async(self, buffer: torch.Tensor, tag: int, op=ReduceOp.SUM, quantize: bool = False) -> AsyncHandle:
        op = ReduceOp.parse(op)
        if not isinstance(buffer, torch.Tensor) or buffer.dim() != 1:
            raise UsageError("buffer must be a one-dimensional tensor")
        if buffer.dtype not in (torch.float32, torch.float64, torch.bfloat16):
            raise UsageError(f"unsupported dtype {buffer.dtype}")
        if not buffer.is_contiguous() or not buffer.is_cuda:
            raise UsageError("buffer must be a contiguous CUDA tensor")
        if quantize and buffer.dtype != torch.float32:
            raise UsageError("quantization requires float32 buffers")
        prev = self._handles.get(tag)
        if prev is not None and prev.pending:
            raise UsageError(f"tag {tag} already has a live operation")
        slot = tag % self.pool_size
        stream = self.streams[slot]
        # the slot stream sees the caller's writes to the buffer
        stream.wait_stream(torch.cuda.current_stream(self.device))
        engine = self.engines[slot]
        self.stats["reduce_attempts"] += 1
        try:
            ticket = engine.all_reduce_async(buffer, op, quantize=quantize, stream=stream)
            handle = AsyncHandle(tag, slot, ticket)
        except UsageError as e:  # disagreement detected at enqueue
            handle = AsyncHandle(tag, slot, None, ReduceResult("aborted", str(e)))
        self._handles[tag] = handle
        return handle

    def await_async_reduce(self, handle: AsyncHandle, timeout: float | None = None) -> ReduceResult:
        if handle._consumed:
            raise UsageError("handle already awaited")
        handle._consumed = True
        if handle._early is not None:
            result = handle._early
        else:
            engine = self.engines[handle.slot]
            try:
                st = engine.await_reduce(handle.ticket)
                result = ReduceResult("completed", "", st.tx_payload_bytes, st.rx_payload_bytes)
            except CollectiveAborted as e:
                result = ReduceResult("aborted", e.reason)
            except UsageError as e:  # parameters disagreed across ranks
                result = ReduceResult("aborted", str(e))
            torch.cuda.current_stream(self.device).wait_stream(self.streams[handle.slot])
        self.stats["reduce_completed" if result.completed else "reduce_aborted"] += 1
        return result

    def all_reduce(self, buffer, tag, op=ReduceOp.SUM, quantize=False) -> ReduceResult:
        return self.await_async_reduce(self.all_reduce_async(buffer, tag, op, quantize))

    def abort(self, tag: int) -> None:
        """ABORT_NOTIFY for `tag` (client.py:196-204): the tag's in-flight
        attempt aborts at its next barrier (or its completion vote) on every
        rank and restores the buffer; ops of other tags queued on the same
        slot are not affected (the abort word is attempt-scoped)."""
        h = self._handles.get(tag)
        if h is not None and h.pending and h.ticket is not None:
            self.engines[h.slot].signal_abort(h.ticket.attempt)

    def restore(self, handle: AsyncHandle, buffer: torch.Tensor) -> None:
        """Completion vetoed (client.py:973-983): hand back the input bytes."""
        self.engines[handle.slot].restore(buffer)

    # -- shared state (client.py:692-798) ----------------------------------
    def sync_shared_state(self, entries: list[SharedStateEntry],
                          strategy: SyncStrategy | str = SyncStrategy.ENFORCE_POPULAR) -> SyncOutcomeResult:
        """Bring every peer to bit-identical entries: GPU digests (one
        multi-entry launch), a plan by the reference's rules, donor->receiver
        copies over NVLink from the donor's memory (IPC), hash verification
        of every fetched entry, and a final digest agreement."""
        if isinstance(strategy, str):
            strategy = SyncStrategy(strategy)
        if any(h.pending for h in self._handles.values()):
            raise UsageError("sync_shared_state while collectives are pending")
        self.stats["sync_calls"] += 1
        torch.cuda.synchronize(self.device)
        hashes = simplehash_many([e.buffer for e in entries])  # HASH #1
        # (key, revision, hash, nbytes, dtype): StateEntryMeta of client.py:705-707
        metas = [(e.key, e.revision, h, e.nbytes, int(e.dtype)) for e, h in zip(entries, hashes)]
        # entries' IPC handles travel with the report so donors need no second round
        handles = []
        for e in entries:
            hb = ctypes.create_string_buffer(64)
            off = ctypes.c_uint64()
            check(lib().pcclb_ipc_handle(e.buffer.data_ptr(), hb, ctypes.byref(off)), "ipc_handle")
            handles.append((bytes(hb.raw), int(off.value)))
        world = dist.get_world_size(self.group)
        reports: list = [None] * world
        dist.all_gather_object(reports, (strategy.value, metas, handles), group=self.group)
        # the master requires the same (key, dtype, nbytes) from every peer (master.py:712)
        shape = [(m[0], m[4], m[3]) for m in metas]
        if any([(m[0], m[4], m[3]) for m in r[1]] != shape for r in reports):
            return SyncOutcomeResult(SyncStatus.ERROR, reason="entry keys, dtypes or sizes differ across peers")
        if all(r[1] == reports[0][1] for r in reports):
            return SyncOutcomeResult(SyncStatus.IN_SYNC)  # no payload moves (SPEC no-op bandwidth)
        plan = select_sync_plan({p: (SyncStrategy(r[0]), r[1]) for p, r in enumerate(reports)})
        if isinstance(plan, str):
            return SyncOutcomeResult(SyncStatus.ERROR, reason=plan)
        me = self.rank
        by_key = {e.key: (i, e) for i, e in enumerate(entries)}
        updated, ok, reason = [], True, ""
        stream = torch.cuda.current_stream(self.device)
        opened = []
        try:
            for key, donor, rev, want in plan[me]:
                i, e = by_key[key]
                # client.py:750-757: never downgrade, never copy a different size
                if rev < e.revision:
                    ok, reason = False, f"plan would downgrade {key!r} from revision {e.revision} to {rev}"
                    break
                if reports[donor][1][i][3] != e.nbytes:
                    ok, reason = False, f"size mismatch for {key!r}"
                    break
                h64, off = reports[donor][2][i]
                ptr = ctypes.c_void_p()
                check(lib().pcclb_ipc_open(ctypes.create_string_buffer(h64, 64), ctypes.byref(ptr)), "ipc_open")
                opened.append(ptr.value)
                check(lib().pcclb_copy(e.buffer.data_ptr(), ptr.value + off, e.nbytes, stream.cuda_stream), "copy")
                e.revision = rev
                updated.append(key)
                self.stats["sync_payload_rx"] += e.nbytes
            if updated:
                got = simplehash_many([by_key[k][1].buffer for k in updated])  # HASH #2 (fetched)
                wants = {k: w for k, _d, _r, w in plan[me]}
                bad = [k for k, h in zip(updated, got) if h != wants[k]]
                if bad:
                    ok, reason = False, f"fetched entries fail verification: {bad}"
            torch.cuda.synchronize(self.device)
        finally:
            dist.barrier(group=self.group)  # donors keep their bytes until every fetch landed
            for p in opened:
                lib().pcclb_ipc_close(p)
        digest = [(e.key, e.revision, h) for e, h in zip(entries, simplehash_many([e.buffer for e in entries]))]
        digests: list = [None] * world
        dist.all_gather_object(digests, (ok, digest), group=self.group)  # SYNC_DONE vote
        if not all(d[0] for d in digests):
            return SyncOutcomeResult(SyncStatus.ERROR, reason=reason or "a peer failed to fetch")
        if any(d[1] != digests[0][1] for d in digests):
            return SyncOutcomeResult(SyncStatus.ERROR, reason="digests differ after sync")
        return SyncOutcomeResult(SyncStatus.UPDATED, updated)
