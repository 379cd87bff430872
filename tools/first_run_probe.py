"""Per-op times of 1 GiB AVG all-reduces over ~10 s (torchrun --nproc-per-node N):
shows whether a fresh box's first multi-GPU process runs slow for a while."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_14065_b200.ring_ipc import DeviceRing, init_from_env  # noqa: E402

rank, world, local = init_from_env("gloo")
dev = torch.device("cuda", local)
n = 1 << 28
buf = torch.randn(n, device=dev)
ring = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, False))
ring.register(buf)
t_start = time.time()
rows = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
while time.time() - t_start < float(sys.argv[1]) if len(sys.argv) > 1 else 10.0:
    torch.distributed.barrier()
    e0.record()
    for _ in range(10):
        ring.run_all_reduce(buf, "avg")
    e1.record()
    torch.cuda.synchronize()
    rows.append((round(time.time() - t_start, 2), round(e0.elapsed_time(e1) / 10, 3)))
if rank == 0:
    print(json.dumps(rows))
ring.close()
