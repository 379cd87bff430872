"""Per-rank body of the multi-GPU ring tests (one process per GPU).

Run as ``python tests/mp_ring_worker.py <world> <port> <outdir> [scenario...]``
by tests/test_ring_ipc_gpu.py through torch.multiprocessing; results are
written to ``<outdir>/rank<r>.json`` and asserted by the parent.
"""

from __future__ import annotations

import json
import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _hash(t) -> int:
    from oracle import simplehash as osh

    return osh.simplehash_c(t.cpu().numpy())


def run(rank: int, world: int, port: int, outdir: str, scenarios: list[str]) -> None:
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    gpu = rank % torch.cuda.device_count()  # >1 rank per GPU only in the oversubscribed W=8 check
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ring as oring
    from paper_2505_14065_b200.collective import CollectiveAborted, UsageError
    from paper_2505_14065_b200.ring_ipc import DeviceRing
    from paper_2505_14065_b200.schedule import payload_bytes
    from tests.golden.gen import RING_CASES, ring_inputs

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        golden = json.load(f)
    dev = torch.device("cuda", gpu)
    out: dict = {"rank": rank, "checks": [], "errors": []}

    def check(name, ok, detail=""):
        out["checks"].append({"name": name, "ok": bool(ok), "detail": str(detail)[:300]})

    try:
        ring = DeviceRing(device=dev, capacity_bytes=64 << 20, timeout_s=20.0)
        rev = None
        if "golden" in scenarios:
            # every golden case with W == world, in identity and reversed ring order
            rev = DeviceRing(device=dev, ring=list(reversed(range(world))), capacity_bytes=64 << 20, timeout_s=20.0)
            # the same cases on the multi-kernel schedule (small path off)
            big = DeviceRing(device=dev, capacity_bytes=64 << 20, timeout_s=20.0, small_max_bytes=0)
            for idx, case in enumerate(RING_CASES):
                w, n, op, quant, dt, seed = case
                if w != world:
                    continue
                want = golden["ring"][idx]["output_hash"]
                inputs = ring_inputs(w, n, np.dtype(dt), seed)
                for eng, tag in ((ring, "id"), (rev, "rev"), (big, "id/multi-kernel")):
                    pos = eng.position
                    buf = torch.from_numpy(inputs[pos].copy()).to(dev)
                    st = eng.run_all_reduce(buf, op, quantize=quant)
                    check(f"golden[{idx}]/{tag} w={w} n={n} {op} q={quant} {dt}", _hash(buf) == want)
                    esz = 1 if quant else np.dtype(dt).itemsize
                    exp = payload_bytes(n, w, esz, pos)
                    check(f"traffic[{idx}]/{tag}", st.tx_payload_bytes == exp and st.rx_payload_bytes == exp,
                          f"{st.tx_payload_bytes} vs {exp}")
        if "faults" in scenarios:
            n = 40_003
            for quant in (False, True):
                # every abort point: the barriers / fused steps and the completion vote
                nb = world + 1 if quant else 3
                for k in range(nb):
                    f = k % world
                    inputs = ring_inputs(world, n, np.dtype("float32"), 500 + k)
                    mine = inputs[ring.position]
                    buf = torch.from_numpy(mine.copy()).to(dev)
                    aborted = False
                    try:
                        ring.run_all_reduce(buf, "sum", quantize=quant, fault_at=k if rank == f else -1)
                    except CollectiveAborted:
                        aborted = True
                    check(f"fault q={quant} at={k} by={f}: aborted", aborted)
                    check(f"fault q={quant} at={k}: restored", buf.cpu().numpy().tobytes() == mine.tobytes())
                    # survivors retry the same op: bit-exact
                    ring.run_all_reduce(buf, "sum", quantize=quant)
                    want = oring.ring_allreduce_chunkwise(inputs, oring.ReduceOp.SUM, quantize=quant)
                    check(f"fault q={quant} at={k}: retry exact", buf.cpu().numpy().tobytes() == want.tobytes())
            # host abort word (the control plane's ABORT_NOTIFY)
            inputs = ring_inputs(world, n, np.dtype("float32"), 900)
            mine = inputs[ring.position]
            buf = torch.from_numpy(mine.copy()).to(dev)
            if rank == world - 1:
                ring.signal_abort()
            aborted = False
            try:
                ring.run_all_reduce(buf, "avg")
            except CollectiveAborted as e:
                aborted = e.source in ("master", "io")
            ring.reset_abort()
            check("host abort: aborted", aborted)
            check("host abort: restored", buf.cpu().numpy().tobytes() == mine.tobytes())
            dist.barrier()
            ring.run_all_reduce(buf, "avg")
            want = oring.ring_allreduce_chunkwise(inputs, oring.ReduceOp.AVG)
            check("host abort: retry exact", buf.cpu().numpy().tobytes() == want.tobytes())
            # abort raised while the attempt runs (after enqueue): the completion vote
            # makes every rank end the same way -- all aborted with their bytes back,
            # or all completed bit-exact
            for qi, quant in enumerate((False, True)):
                inputs = ring_inputs(world, (1 << 20) + 17, np.dtype("float32"), 903 + qi)
                mine = inputs[ring.position]
                buf = torch.from_numpy(mine.copy()).to(dev)
                t = ring.all_reduce_async(buf, "avg", quantize=quant)
                if rank == world - 1:
                    ring.signal_abort(t.attempt)
                try:
                    ring.await_reduce(t)
                    outcome = "completed"
                except CollectiveAborted:
                    outcome = "aborted"
                outs = [None] * world
                dist.all_gather_object(outs, outcome)
                check(f"mid-op abort q={quant}: same outcome everywhere", len(set(outs)) == 1, outs)
                want = mine if outcome == "aborted" else oring.ring_allreduce_chunkwise(inputs, oring.ReduceOp.AVG, quant)
                check(f"mid-op abort q={quant}: bytes ({outcome})", buf.cpu().numpy().tobytes() == want.tobytes())
            # non-finite under quantization: everyone aborts and restores
            inputs = ring_inputs(world, n, np.dtype("float32"), 901)
            inputs[world // 2][77] = np.inf
            mine = inputs[ring.position]
            buf = torch.from_numpy(mine.copy()).to(dev)
            aborted = False
            try:
                ring.run_all_reduce(buf, "sum", quantize=True)
            except CollectiveAborted:
                aborted = True
            check("nonfinite: aborted", aborted)
            check("nonfinite: restored", buf.cpu().numpy().tobytes() == mine.tobytes())
            # several attempts in flight (all_reduce_async), awaited afterwards
            sets = [ring_inputs(world, 10_007 + 13 * i, np.dtype("float32"), 950 + i) for i in range(3)]
            bufs = [torch.from_numpy(x[ring.position].copy()).to(dev) for x in sets]
            tickets = [ring.all_reduce_async(b, "avg", quantize=(i == 1)) for i, b in enumerate(bufs)]
            for i, (t, b, x) in enumerate(zip(tickets, bufs, sets)):
                ring.await_reduce(t)
                want = oring.ring_allreduce_chunkwise(x, oring.ReduceOp.AVG, quantize=(i == 1))
                check(f"async in flight [{i}]", b.cpu().numpy().tobytes() == want.tobytes())
            # completion veto restore (client.py:973-983)
            inputs = ring_inputs(world, n, np.dtype("float64"), 902)
            mine = inputs[ring.position]
            buf = torch.from_numpy(mine.copy()).to(dev)
            ring.run_all_reduce(buf, "max")
            ring.restore(buf)
            check("veto restore", buf.cpu().numpy().tobytes() == mine.tobytes())
        if "registered" in scenarios:
            # zero-copy path: peers read the registered buffer in place (the
            # one-kernel small path always copies in, so it is off here)
            ring.set_small_max_bytes(0)
            n = (1 << 22) + 5
            inputs = [np.random.default_rng(300 + p).normal(0, 2, n).astype(np.float32) for p in range(world)]
            reg = torch.empty(n + 64, dtype=torch.float32, device=dev)
            ring.register(reg)
            for lo_off, cnt, quant, op in ((0, n, False, "avg"), (7, n - 100, False, "sum"), (3, n - 9, True, "avg"), (0, 1000, False, "max")):
                view = reg[lo_off : lo_off + cnt]
                mine = inputs[ring.position][:cnt]
                view.copy_(torch.from_numpy(mine))
                ring.run_all_reduce(view, op, quantize=quant)
                want = oring.ring_allreduce_chunkwise([x[:cnt] for x in inputs], oring.ReduceOp[op.upper()], quantize=quant)
                check(f"registered off={lo_off} n={cnt} q={quant} {op}", view.cpu().numpy().tobytes() == want.tobytes())
            # abort atomicity in zero-copy mode: barriers 0, 1 and the completion
            # vote (2), which also waits until every peer's pushes into this
            # rank's buffer landed before the restore
            for k in range(3):
                view = reg[:n]
                mine = inputs[ring.position]
                view.copy_(torch.from_numpy(mine))
                aborted = False
                try:
                    ring.run_all_reduce(view, "sum", fault_at=k if rank == k % world else -1)
                except CollectiveAborted:
                    aborted = True
                check(f"registered fault at={k}: aborted", aborted)
                check(f"registered fault at={k}: restored", view.cpu().numpy().tobytes() == mine.tobytes())
            # completion veto restore in zero-copy mode (backup fused into the gather)
            view = reg[5 : 5 + n - 50]
            mine = inputs[ring.position][: n - 50]
            view.copy_(torch.from_numpy(mine))
            ring.run_all_reduce(view, "avg")
            ring.restore(view)
            check("registered veto restore", view.cpu().numpy().tobytes() == mine.tobytes())
            # one rank unregistered -> every rank rejects the op, buffers intact
            other = torch.from_numpy(inputs[ring.position].copy()).to(dev)
            target = other if rank == 0 else reg[:n]
            target.copy_(torch.from_numpy(inputs[ring.position]))
            rejected = False
            try:
                ring.run_all_reduce(target, "sum")
            except (UsageError, CollectiveAborted):  # a rank may see a peer's abort token first
                rejected = True
            check("registration mismatch rejected", rejected)
            check("registration mismatch intact", target.cpu().numpy().tobytes() == inputs[ring.position].tobytes())
            ring.set_small_max_bytes(None)
            ring.deregister(0)
        if "qedge" in scenarios:
            # quantized schedule variants: fused at 3 and 4 CTAs/SM (slots 2, 1) and the
            # barrier-per-step fallback (slots 5); misaligned views, chunks shorter than
            # a ready-flag block, sizes straddling block boundaries, every op
            cases = [(1, 0, "sum"), (world - 1, 1, "avg"), (7, 1, "max"), (65536 * world + 5, 1, "min"),
                     (3 * 65536 * world + 17, 3, "avg"), ((1 << 20) + 3, 0, "sum"),
                     (2 * 262144 * world + 9, 2, "avg"), (262144 * world - 1, 0, "max")]
            for slots in (2, 1, 5):
                eng = DeviceRing(device=dev, capacity_bytes=64 << 20, timeout_s=20.0, slots=slots)
                for ci, (n, off, op) in enumerate(cases):
                    inputs = ring_inputs(world, n, np.dtype("float32"), 700 + ci)
                    base = torch.zeros(n + 8, device=dev)
                    view = base[off:off + n]
                    view.copy_(torch.from_numpy(inputs[eng.position]))
                    eng.run_all_reduce(view, op, quantize=True)
                    want = oring.ring_allreduce_chunkwise(inputs, getattr(oring.ReduceOp, op.upper()), quantize=True)
                    check(f"qedge slots={slots} n={n} off={off} {op}", view.cpu().numpy().tobytes() == want.tobytes())
                    check(f"qedge slots={slots} n={n}: guard bytes", float(base[:off].abs().sum()) == 0.0
                          and float(base[off + n:].abs().sum()) == 0.0)
                eng.close()
            # ranks on different quantized schedules (rank 0 on the barrier fallback)
            # must reject the op together and keep their bytes
            eng = DeviceRing(device=dev, capacity_bytes=64 << 20, timeout_s=20.0, slots=5 if rank == 0 else 2)
            inputs = ring_inputs(world, 10_001, np.dtype("float32"), 790)
            buf = torch.from_numpy(inputs[eng.position].copy()).to(dev)
            rejected = False
            try:
                eng.run_all_reduce(buf, "avg", quantize=True)
            except (UsageError, CollectiveAborted):
                rejected = True
            check("qedge: schedule mismatch rejected", rejected)
            check("qedge: schedule mismatch intact", buf.cpu().numpy().tobytes() == inputs[eng.position].tobytes())
            eng.close()
        if "ext" in scenarios:
            # PROD extension (parity unpinned: oracle/ring.py's np.multiply fold)
            multi = DeviceRing(device=dev, capacity_bytes=64 << 20, timeout_s=20.0, small_max_bytes=0)
            for n in (1, 4099, 300_007):
                g_ = np.random.default_rng(n)
                inputs = [(1.0 + 0.05 * g_.normal(0, 1, n)).astype(np.float32) for _ in range(world)]
                for eng, tag in ((ring, "small"), (multi, "multi-kernel")):
                    for quant in (False, True):
                        buf = torch.from_numpy(inputs[eng.position].copy()).to(dev)
                        eng.run_all_reduce(buf, "prod", quantize=quant)
                        want = oring.ring_allreduce_chunkwise(inputs, oring.ReduceOp.PROD, quantize=quant)
                        check(f"PROD {tag} n={n} q={quant}", buf.cpu().numpy().tobytes() == want.tobytes())
            # bf16 extension (oracle/bf16.py): small path and multi-kernel schedule
            from oracle import bf16 as ob

            for n in (1, 4099, 300_007):
                g_ = np.random.default_rng(n + 5)
                inputs = [ob.from_f32(g_.normal(0, 1, n).astype(np.float32)) for _ in range(world)]
                for eng, tag in ((ring, "small"), (multi, "multi-kernel")):
                    for op in ("avg", "max"):
                        buf = torch.from_numpy(inputs[eng.position].view(np.int16).copy()).to(dev).view(torch.bfloat16)
                        eng.run_all_reduce(buf, op)
                        want = ob.ring_allreduce_chunkwise(inputs, oring.ReduceOp[op.upper()])
                        got = buf.view(torch.int16).cpu().numpy().view(np.uint16)
                        check(f"bf16 {tag} n={n} {op}", got.tobytes() == want.tobytes())
            multi.close()
        if "large" in scenarios or "large_small" in scenarios:
            n = (1 << 24) + 3 if "large" in scenarios else (1 << 21) + 3
            for quant in (False, True):
                inputs = [np.random.default_rng(70 + p).normal(0, 1, n).astype(np.float32) for p in range(world)]
                buf = torch.from_numpy(inputs[ring.position].copy()).to(dev)
                ring.run_all_reduce(buf, "avg", quantize=quant)
                got = buf.cpu().numpy()
                # each rank verifies its owned chunk and one other chunk against the oracle
                bounds = oring.chunk_bounds(n, world)
                for c in {(ring.position + 1) % world, ring.position}:
                    lo, hi = bounds[c]
                    spans = [inputs[(c + k) % world][lo:hi] for k in range(world)]
                    want = oring.reduce_chunk(spans, oring.ReduceOp.AVG, quant, world)
                    check(f"large q={quant} chunk {c}", got[lo:hi].tobytes() == want.tobytes())
                hs = [None] * world
                dist.all_gather_object(hs, _hash(buf))
                check(f"large q={quant}: identical on all ranks", len(set(hs)) == 1)
        for sc in scenarios:
            if not sc.startswith("death_"):
                continue
            # a peer process dies while the attempt runs (its kernels in flight,
            # its workspace mapped by the survivors): the survivors end the
            # attempt the same way (aborted with their bytes back, or completed
            # if the victim's vote landed first), keep a healthy CUDA context,
            # and retry at W-1 on a new ring (test_cluster.py:256-307)
            import time

            quant = sc == "death_quant"
            victim = world - 1
            survivors = [r for r in range(world) if r != victim]
            sub = dist.new_group(survivors, backend="gloo")  # before anyone dies
            n = 300_000_007
            eng = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, quant), timeout_s=5.0)
            g = torch.Generator(device=dev).manual_seed(60 + rank)
            src = torch.randn(n, generator=g, device=dev) * (1e-2 if quant else 1.0)
            buf = src.clone()
            torch.cuda.synchronize()
            dist.barrier()
            if rank == 0:
                # the victim arrives at barrier 0 (its token is visible to every
                # peer) and spins there; it dies before this rank arrives, so the
                # others pass the barrier and then read the dead rank's workspace
                time.sleep(0.5)
            t = eng.all_reduce_async(buf, "sum", quantize=quant)
            if rank == victim:
                time.sleep(0.05)
                with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
                    json.dump(out, f)
                os._exit(0)  # no cleanup: the context dies with the kernels in flight
            try:
                eng.await_reduce(t)
                outcome = "completed"
            except CollectiveAborted:
                outcome = "aborted"
            outs = [None] * len(survivors)
            dist.all_gather_object(outs, outcome, group=sub)
            check(f"{sc}: survivors agree ({outs})", len(set(outs)) == 1, outs)
            if outcome == "aborted":
                check(f"{sc}: restored", bool(torch.equal(buf, src)))
            # the context is healthy: new work runs and the old engine closes
            x = torch.arange(1000, device=dev, dtype=torch.float64).sum().item()
            check(f"{sc}: context healthy", x == 499500.0, x)
            try:
                eng.close()
            except Exception as exc:  # noqa: BLE001
                check(f"{sc}: old engine closes", False, exc)
            # retry at W-1 on a new ring over the survivors, bit-exact
            buf.copy_(src)
            m = 1_000_003
            part = buf[:m]
            eng2 = DeviceRing(group=sub, device=dev, capacity_bytes=64 << 20, timeout_s=20.0)
            eng2.run_all_reduce(part, "sum", quantize=quant)
            ins = []
            for r_ in survivors:
                g2 = torch.Generator(device=dev).manual_seed(60 + r_)
                ins.append((torch.randn(n, generator=g2, device=dev) * (1e-2 if quant else 1.0))[:m].cpu().numpy())
            want = oring.ring_allreduce_chunkwise(ins, oring.ReduceOp.SUM, quantize=quant)
            check(f"{sc}: retry at W-1 exact", part.cpu().numpy().tobytes() == want.tobytes())
            eng2.close()
            with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
                json.dump(out, f)
            os._exit(0)  # the default group has a dead member: skip its teardown
        if "config" in scenarios:
            # BASELINE config sizes; inputs generated on the device from per-rank
            # seeds, so any rank can regenerate a peer's chunk for the oracle
            def gen(p, n, scale, seed):
                gen_ = torch.Generator(device=dev).manual_seed(seed + p)
                return torch.randn(n, generator=gen_, device=dev) * scale

            big = DeviceRing(device=dev, capacity_bytes=2 << 30, timeout_s=60.0)
            for tag, n, quant, scale in (("config2 plain AVG", 268_435_456, False, 1.0),
                                         ("config3-chunk u8 AVG", 150_000_000 * world, True, 1e-2)):
                seed = 4000 if not quant else 5000
                buf = gen(big.position, n, scale, seed)
                big.run_all_reduce(buf, "avg", quantize=quant)
                torch.cuda.synchronize()
                bounds = oring.chunk_bounds(n, world)
                for c in sorted({big.position, (big.position + 1) % world}):
                    lo, hi = bounds[c]
                    spans = [gen((c + k) % world, n, scale, seed)[lo:hi].cpu().numpy() for k in range(world)]
                    want = oring.reduce_chunk(spans, oring.ReduceOp.AVG, quant, world)
                    check(f"{tag} chunk {c} ({hi - lo} elems)", buf[lo:hi].cpu().numpy().tobytes() == want.tobytes())
                    del spans, want
                hs = [None] * world
                dist.all_gather_object(hs, _hash(buf))
                check(f"{tag}: identical on all ranks", len(set(hs)) == 1)
                del buf
                torch.cuda.empty_cache()
            big.close()
        ring.close()
        if rev is not None:
            rev.close()
            big.close()
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
    scenarios = sys.argv[4:] or ["golden", "faults", "registered", "qedge", "ext", "large"]
    mp.spawn(_entry, args=(world, port, outdir, scenarios), nprocs=world, join=True)
