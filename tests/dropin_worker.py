"""One peer of the drop-in test (tests/test_dropin_reference_gpu.py): the
UNMODIFIED reference client (churncomm from baseline/_ref, installed from
/root/reference with pip) joins the reference MasterServer over TCP; only its
engine seam -- ``churncomm.client.run_all_reduce`` (client.py:932 ->
collective.py:489) -- is rebound to the NVLink engine as in
INTEGRATION.md §3. Init votes, the committed ring, seq numbers, the complete
vote and the veto restore all run through the reference's own control plane.

usage: python tests/dropin_worker.py <rank> <world> <master_port> <dist_port> <outdir>
"""

from __future__ import annotations

import json
import os
import sys
import threading
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(1, os.path.join(ROOT, "baseline", "_ref"))


def main(rank: int, world: int, master_port: int, dist_port: int, outdir: str) -> None:
    import torch
    import torch.distributed as dist

    out = {"rank": rank, "checks": [], "errors": []}

    def check(name, ok, detail=""):
        out["checks"].append({"name": name, "ok": bool(ok), "detail": str(detail)[:300]})

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(dist_port)
        gpu = rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        dev = torch.device("cuda", gpu)
        dist.init_process_group("gloo", rank=rank, world_size=world)

        import churncomm.client as rclient
        from churncomm.collective import CollectiveAborted as RefAborted
        from churncomm.collective import ReduceOp as RefOp
        from churncomm.config import ClientConfig

        from oracle import ring as oring
        from paper_2505_14065_b200.collective import CollectiveAborted
        from paper_2505_14065_b200.ring_ipc import DeviceRing

        # join in rank order so peer ids are deterministic (the first peer is
        # accepted alone), then every peer runs topology rounds until the
        # veterans' vote admits the newcomers (the reference's grow_world)
        comm = None
        for r in range(world):
            if r == rank:
                comm = rclient.connect(config=ClientConfig(master_addr=f"127.0.0.1:{master_port}", pool_size=1,
                                                           probe_bytes=64 * 1024, vote_timeout=15.0))
                if r == 0:
                    comm.update_topology()
            dist.barrier()
        for _ in range(200):
            res = comm.update_topology()
            if res.accepted and res.world == world:
                break
            time.sleep(0.02)
        check("reference master admitted every peer", comm.get_world_size() == world, comm.get_world_size())
        ids = [None] * world
        dist.all_gather_object(ids, comm.peer_id)
        rank_of = {pid: r for r, pid in enumerate(ids)}

        engines: dict = {}
        lock = threading.Lock()

        def gpu_run_all_reduce(ctx, sender, backup):
            """The engine seam: same contract as collective.run_all_reduce --
            reduce ctx.buffer in place in the committed ring's order, or raise
            CollectiveAborted after restoring it (collective.py:568-574)."""
            ring = [rank_of[p] for p in comm.view.ring]
            if ring.index(rank) != ctx.rank:
                raise RefAborted("ring view differs from the commit", source="io")
            key = tuple(ring)
            with lock:
                if key not in engines:  # collective: every peer's first op on this ring
                    engines[key] = DeviceRing(ring=ring, device=dev, capacity_bytes=64 << 20, timeout_s=20.0)
            eng = engines[key]
            t = torch.from_numpy(ctx.buffer).to(dev)
            # ABORT_NOTIFY -> the attempt-scoped abort word (client.py:196-204)
            watcher_stop = threading.Event()

            def watch():
                while not watcher_stop.is_set():
                    if ctx.abort_event.wait(0.01):
                        eng.signal_abort()
                        return

            th = threading.Thread(target=watch, daemon=True)
            th.start()
            try:
                st = eng.run_all_reduce(t, ctx.op.name.lower(), quantize=ctx.quantize)
            except CollectiveAborted as e:
                raise RefAborted(e.reason, source=e.source) from None
            finally:
                watcher_stop.set()
            ctx.buffer[...] = t.cpu().numpy()
            ctx.tx_payload_bytes = st.tx_payload_bytes
            ctx.rx_payload_bytes = st.rx_payload_bytes

        rclient.run_all_reduce = gpu_run_all_reduce  # the only change to the reference

        # config 1: 2-peer SUM of 1 M f32 (BASELINE configs[0]); then u8 AVG
        n = 1 << 20
        cases = [("config1 SUM", RefOp.SUM, False, 1), ("u8 AVG", RefOp.AVG, True, 2), ("MAX", RefOp.MAX, False, 3)]
        for name, op, quant, tag in cases:
            inputs = [np.random.default_rng(r + 10 * tag).normal(0, 1, n).astype(np.float32) for r in range(world)]
            buf = inputs[rank].copy()
            result = comm.all_reduce(buf, tag=tag, op=op, quantize=quant)
            check(f"{name}: completed through the reference master", result.status == "completed", result)
            ring = [rank_of[p] for p in comm.view.ring]
            want = oring.ring_allreduce_chunkwise([inputs[g] for g in ring], oring.ReduceOp[op.name], quantize=quant)
            check(f"{name}: bit-exact vs oracle in the committed ring order {ring}", buf.tobytes() == want.tobytes())
            check(f"{name}: traffic in the complete vote", result.tx_bytes > 0 and result.tx_bytes == result.rx_bytes,
                  (result.tx_bytes, result.rx_bytes))
        for eng in engines.values():
            eng.close()
        comm.close()
    except Exception:  # noqa: BLE001
        out["errors"].append(traceback.format_exc())
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
