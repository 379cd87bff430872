"""Per-phase device times of the NVLink ring (PCCLB_RING_PROFILE=1).

torchrun --nproc-per-node N tools/ring_phases.py [elems] [quant]"""
import json
import os
import sys

os.environ["PCCLB_RING_PROFILE"] = "1"
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_14065_b200.ring_ipc import DeviceRing, init_from_env  # noqa: E402

rank, world, local = init_from_env("gloo")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
quant = len(sys.argv) > 2 and sys.argv[2] == "quant"
op = sys.argv[3] if len(sys.argv) > 3 else "avg"
dev = torch.device("cuda", local)
buf = torch.randn(n, device=dev) * (1e-2 if quant else 1)
ring = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, quant))
if os.environ.get("REGISTER", "1") == "1":
    ring.register(buf)
rows = []
for i in range(8):
    st = ring.run_all_reduce(buf, op, quantize=quant)
    if i >= 3:
        rows.append(st.phase_ms)
avg = [round(sum(r[k] for r in rows) / len(rows), 4) for k in range(len(rows[0]))]
allr = [None] * world
torch.distributed.all_gather_object(allr, avg)
if rank == 0:
    print(json.dumps({"world": world, "n": n, "quant": quant, "phase_ms_per_rank": allr, "total_ms": [round(sum(a), 3) for a in allr]}))
ring.close()
