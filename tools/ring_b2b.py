"""Back-to-back NVLink all-reduces: per-op device time from events between
enqueues, and host enqueue time. torchrun --nproc-per-node N tools/ring_b2b.py [elems]"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_14065_b200.ring_ipc import DeviceRing, init_from_env  # noqa: E402

rank, world, local = init_from_env("gloo")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
dev = torch.device("cuda", local)
buf = torch.randn(n, device=dev)
ring = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, False))
if os.environ.get("REGISTER", "1") == "1":
    ring.register(buf)
for _ in range(3):
    ring.run_all_reduce(buf, "avg")
torch.cuda.synchronize()
torch.distributed.barrier()
K = 10
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
host = []
tickets = []
s = torch.cuda.current_stream()
for k in range(K):
    ev[k].record(s)
    t0 = time.perf_counter()
    tickets.append(ring.all_reduce_async(buf, "avg"))
    host.append((time.perf_counter() - t0) * 1e3)
ev[K].record(s)
for t in tickets:
    ring.await_reduce(t)
torch.cuda.synchronize()
per = [round(ev[k].elapsed_time(ev[k + 1]), 4) for k in range(K)]
allr = [None] * world
torch.distributed.all_gather_object(allr, {"gpu_ms": per, "host_enqueue_ms": [round(h, 3) for h in host]})
if rank == 0:
    print(json.dumps({"world": world, "n": n, "per_rank": allr}))
ring.close()
