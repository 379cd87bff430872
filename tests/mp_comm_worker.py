"""Per-rank body of the Communicator tests (one process per GPU):
API usage errors, concurrent tags, parameter disagreement, shared-state sync
(config 4: one drifted peer; a newcomer), and churn (config 5: two concurrent
quantized all-reduces, one peer dropped mid-way, retry at W-1, rejoin)."""

from __future__ import annotations

import json
import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def run(rank: int, world: int, port: int, outdir: str, scenarios: list[str]) -> None:
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    gpu = rank % torch.cuda.device_count()  # oversubscribed (same-device IPC) when GPUs < world
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ring as oring
    from oracle import simplehash as osh
    from paper_2505_14065_b200.collective import UsageError
    from paper_2505_14065_b200.communicator import Communicator, SyncStatus
    from paper_2505_14065_b200.ring_ipc import DeviceRing
    from paper_2505_14065_b200.sharedstate import DType, SharedStateEntry

    dev = torch.device("cuda", gpu)
    out: dict = {"rank": rank, "checks": [], "errors": []}

    def check(name, ok, detail=""):
        out["checks"].append({"name": name, "ok": bool(ok), "detail": str(detail)[:300]})

    def inputs(n, seed, w=world, scale=1.0):
        return [np.random.default_rng(seed + p).normal(0, scale, n).astype(np.float32) for p in range(w)]

    try:
        if "api" in scenarios:
            comm = Communicator(device=dev, pool_size=2, timeout_s=20.0)
            check("world size", comm.get_world_size() == world)
            # usage errors before any native call (client.py:812-824, test_bindings.py:64-80)
            for bad, what in ((torch.zeros(4, 4, device=dev), "2-D"), (torch.zeros(8, dtype=torch.int32, device=dev), "int"),
                              (torch.zeros(8, dtype=torch.float64, device=dev), "quant f64")):
                try:
                    comm.all_reduce_async(bad, 5, "sum", quantize=(what == "quant f64"))
                    check(f"usage error {what}", False)
                except UsageError:
                    check(f"usage error {what}", True)
            # two tags in flight on two slots: plain AVG (tag 0) and u8 AVG (tag 1)
            x0, x1 = inputs(100_003, 10), inputs(77_777, 20, scale=1e-2)
            b0 = torch.from_numpy(x0[rank].copy()).to(dev)
            b1 = torch.from_numpy(x1[rank].copy()).to(dev)
            h0 = comm.all_reduce_async(b0, 0, "avg")
            h1 = comm.all_reduce_async(b1, 1, "avg", quantize=True)
            try:
                comm.all_reduce_async(b0, 0, "avg")
                check("tag busy", False)
            except UsageError:
                check("tag busy", True)
            r1 = comm.await_async_reduce(h1)
            r0 = comm.await_async_reduce(h0)
            check("tag0 completed", r0.completed, r0)
            check("tag1 completed", r1.completed, r1)
            check("tag0 exact", b0.cpu().numpy().tobytes() == oring.ring_allreduce_chunkwise(x0, oring.ReduceOp.AVG).tobytes())
            check("tag1 exact", b1.cpu().numpy().tobytes() == oring.ring_allreduce_chunkwise(x1, oring.ReduceOp.AVG, True).tobytes())
            check("traffic identity", abs(r0.tx_bytes - 2 * (world - 1) / world * 100_003 * 4) <= 0.01 * r0.tx_bytes)
            # parameter disagreement: one rank reduces a different count -> everyone aborts, bytes intact
            n = 5000 + (1 if rank == 0 else 0)
            x = np.random.default_rng(rank).normal(0, 1, n).astype(np.float32)
            b = torch.from_numpy(x.copy()).to(dev)
            r = comm.all_reduce(b, 2, "sum")
            check("param mismatch aborted", not r.completed, r)
            check("param mismatch intact", b.cpu().numpy().tobytes() == x.tobytes())
            # non-finite under quantization (client.py:871-873): aborted, intact
            x = np.random.default_rng(rank + 9).normal(0, 1, 4096).astype(np.float32)
            if rank == world - 1:
                x[17] = np.nan
            b = torch.from_numpy(x.copy()).to(dev)
            r = comm.all_reduce(b, 3, "sum", quantize=True)
            check("nonfinite aborted", not r.completed, r)
            check("nonfinite intact", b.cpu().numpy().tobytes() == x.tobytes())
            comm.close()

        if "sync" in scenarios:
            comm = Communicator(device=dev, pool_size=1, timeout_s=20.0)
            shapes = [(1283, 64), (64, 64), (16, 64), (143, 64), (64,), (2048,)]

            def state(seed):
                g = np.random.default_rng(seed)
                return [torch.from_numpy(g.normal(0, 1, int(np.prod(s))).astype(np.float32)).to(torch.bfloat16).to(dev)
                        for s in shapes]

            tensors = state(1234)
            if rank == 1 % world:  # the drifted peer: one bit flipped at equal revision
                tensors[2].view(torch.uint8)[77] ^= 1
            entries = [SharedStateEntry(f"w{i}", DType.U8, t.view(torch.uint8), revision=7) for i, t in enumerate(tensors)]
            before = [osh.simplehash_c(e.buffer.cpu().numpy()) for e in entries]
            res = comm.sync_shared_state(entries)
            check("drift: updated", res.status is SyncStatus.UPDATED, res)
            clean = [osh.simplehash_c(t.view(torch.uint8).cpu().numpy()) for t in state(1234)]
            got = [osh.simplehash_c(e.buffer.cpu().numpy()) for e in entries]
            alls = [None] * world
            dist.all_gather_object(alls, got)
            check("drift: digest parity", all(a == got for a in alls))
            if world >= 3:  # the majority's bytes win (with two peers the smaller hash does)
                check("drift: popular state everywhere", got == clean)
            else:
                pre = [None] * world
                dist.all_gather_object(pre, before)
                check("drift: tie -> smaller hash wins", got[2] == min(p[2] for p in pre))
            fetched = comm.stats["sync_payload_rx"]
            res = comm.sync_shared_state(entries)
            check("second sync is a no-op", res.status is SyncStatus.IN_SYNC and comm.stats["sync_payload_rx"] == fetched, res)
            ref = got
            # newcomer at revision 0 with other contents takes everything
            if rank == world - 1:
                for e, t in zip(entries, state(999)):
                    e.buffer.copy_(t.view(torch.uint8))
                    e.revision = 0
            res = comm.sync_shared_state(entries)
            check("newcomer: updated", res.status is SyncStatus.UPDATED, res)
            check("newcomer: state", [osh.simplehash_c(e.buffer.cpu().numpy()) for e in entries] == ref)
            check("newcomer: revision", all(e.revision == 7 for e in entries))
            # one peer's entry has another size under the same key: every peer
            # reports an error and nobody copies (master.py:712, client.py:750-757)
            n_odd = 4096 + (64 if rank == 0 else 0)
            odd = torch.zeros(n_odd, dtype=torch.uint8, device=dev) + rank
            res = comm.sync_shared_state([SharedStateEntry("odd", DType.U8, odd, revision=1 + rank)])
            check("size mismatch: error", res.status is SyncStatus.ERROR, res)
            check("size mismatch: untouched", bool((odd == rank).all()))
            comm.close()

        if "sync_scale" in scenarios:
            # config 4 at size: every rank holds the 16.06 GB Llama-3-8B-like state;
            # the drifted peer has one flipped bit in the 1.05 GB embedding at equal
            # revision; one sync restores bit parity (a single entry moves)
            import time

            from bench import llama3_8b_layout

            layout = llama3_8b_layout()
            total = sum(n_ for _, n_ in layout)
            state = torch.empty(total, dtype=torch.bfloat16, device=dev)
            gen = torch.Generator(device=dev).manual_seed(77)
            state.view(torch.int16).random_(-32768, 32767, generator=gen)
            views, off = [], 0
            for _, n_ in layout:
                views.append(state[off: off + n_])
                off += n_
            from paper_2505_14065_b200 import simplehash_many

            clean = simplehash_many(views)  # digests before the drift
            drifted = 1 % world
            if rank == drifted:
                views[0].view(torch.int16)[12345] ^= 1
            entries = [SharedStateEntry(name, DType.U8, v.view(torch.uint8), revision=3)
                       for (name, _), v in zip(layout, views)]
            comm = Communicator(device=dev, pool_size=1, timeout_s=60.0)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            res = comm.sync_shared_state(entries)
            dt = time.perf_counter() - t0
            if world >= 3:
                check("sync 16 GB: updated", res.status in (SyncStatus.UPDATED,), res)
                check("sync 16 GB: popular state everywhere", simplehash_many(views) == clean)
                check("sync 16 GB: one entry moved", rank != drifted or comm.stats["sync_payload_rx"] == views[0].numel() * 2,
                      comm.stats["sync_payload_rx"])
            else:  # two peers: the smaller hash wins the tie
                got = simplehash_many(views)
                alls = [None] * world
                dist.all_gather_object(alls, got)
                check("sync 16 GB: digest parity", all(a == got for a in alls))
            check(f"sync 16 GB: {dt:.2f} s host time", dt < 30.0, dt)
            comm.close()
            del state, views, entries
            torch.cuda.empty_cache()

        if "churn_scale" in scenarios and world >= 3:
            # config 5 at size: two concurrent u8 AVG all-reduces of 600 M f32 each
            # (tags 0 and 1); the dropped peer never enqueues tag 1: tag 0 completes
            # bit-exact (own chunk against the oracle), tag 1 aborts and restores
            n = 600_000_000
            comm = Communicator(device=dev, pool_size=2, timeout_s=10.0,
                                capacity_bytes=DeviceRing.required_bytes(n, world, 4, True))

            def gen_(p, seed):
                g_ = torch.Generator(device=dev).manual_seed(seed + p)
                return torch.randn(n, generator=g_, device=dev) * 1e-2

            b0, b1 = gen_(rank, 100), gen_(rank, 200)
            src1 = b1.clone()
            dropped = world - 1
            torch.cuda.synchronize()
            dist.barrier()
            h0 = comm.all_reduce_async(b0, 0, "avg", quantize=True)
            if rank != dropped:
                h1 = comm.all_reduce_async(b1, 1, "avg", quantize=True)
            r0 = comm.await_async_reduce(h0)
            check("churn 600M: tag0 completed", r0.completed, r0)
            bounds = oring.chunk_bounds(n, world)
            c = (rank + 1) % world
            lo, hi = bounds[c]
            spans = [gen_((c + k) % world, 100)[lo:hi].cpu().numpy() for k in range(world)]
            want = oring.reduce_chunk(spans, oring.ReduceOp.AVG, True, world)
            check("churn 600M: tag0 own chunk exact", b0[lo:hi].cpu().numpy().tobytes() == want.tobytes())
            del spans, want
            if rank != dropped:
                r1 = comm.await_async_reduce(h1)
                check("churn 600M: tag1 aborted", not r1.completed, r1)
                check("churn 600M: tag1 restored", bool(torch.equal(b1, src1)))
            comm.close()
            dist.barrier()

        if "churn" in scenarios and world >= 3:
            # config 5: tags 0 and 1 (two halves of a pseudo-gradient), u8 AVG, in flight together
            comm = Communicator(device=dev, pool_size=2, timeout_s=3.0)
            n = 250_001
            d0, d1 = inputs(n, 100, scale=1e-2), inputs(n, 200, scale=1e-2)
            b0 = torch.from_numpy(d0[rank].copy()).to(dev)
            b1 = torch.from_numpy(d1[rank].copy()).to(dev)
            dropped = world - 1
            h0 = comm.all_reduce_async(b0, 0, "avg", quantize=True)
            if rank != dropped:  # the dropped peer dies before tag 1 reaches the wire
                h1 = comm.all_reduce_async(b1, 1, "avg", quantize=True)
            r0 = comm.await_async_reduce(h0)
            check("churn: tag0 completed", r0.completed, r0)
            check("churn: tag0 exact at W", b0.cpu().numpy().tobytes()
                  == oring.ring_allreduce_chunkwise(d0, oring.ReduceOp.AVG, True).tobytes())
            if rank != dropped:
                r1 = comm.await_async_reduce(h1)
                check("churn: tag1 aborted", not r1.completed, r1)
                check("churn: tag1 restored", b1.cpu().numpy().tobytes() == d1[rank].tobytes())
            comm.close()
            survivors = [r for r in range(world) if r != dropped]
            sub = dist.new_group(survivors, backend="gloo")
            if rank != dropped:
                # the survivors retry tag 1 at W-1 in the new (reversed) ring order
                ring_order = list(reversed(range(len(survivors))))
                c2 = Communicator(group=sub, device=dev, pool_size=2, ring=ring_order, timeout_s=20.0)
                r1 = c2.all_reduce(b1, 1, "avg", quantize=True)
                check("churn: retry completed", r1.completed, r1)
                pos = ring_order.index(survivors.index(rank))
                order = [d1[survivors[g]] for g in ring_order]
                want = oring.ring_allreduce(order, oring.ReduceOp.AVG, quantize=True)[pos]
                check("churn: retry exact at W-1", b1.cpu().numpy().tobytes() == want.tobytes())
                c2.close()
            dist.barrier()
            # rejoin: the returning peer syncs the survivors' state (two buffers) and all digests agree
            comm = Communicator(device=dev, pool_size=1, timeout_s=20.0)
            rev = 1 if rank != dropped else 0
            entries = [SharedStateEntry("delta0", DType.F32, b0, revision=rev), SharedStateEntry("delta1", DType.F32, b1, revision=rev)]
            res = comm.sync_shared_state(entries)
            check("rejoin: updated", res.status is SyncStatus.UPDATED, res)
            hs = [None] * world
            dist.all_gather_object(hs, [osh.simplehash_c(e.buffer.cpu().numpy()) for e in entries])
            check("rejoin: digest parity", all(h == hs[0] for h in hs), hs)
            comm.close()
    except Exception:  # noqa: BLE001
        out["errors"].append(traceback.format_exc())
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(out, f)
    try:
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        pass


def _entry(rank, world, port, outdir, scenarios):
    run(rank, world, port, outdir, scenarios)


if __name__ == "__main__":
    import torch.multiprocessing as mp

    world, port, outdir = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    scenarios = sys.argv[4:] or ["api", "sync", "churn"]
    mp.spawn(_entry, args=(world, port, outdir, scenarios), nprocs=world, join=True)
