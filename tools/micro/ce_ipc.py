"""Copy-engine peer copy through CUDA IPC mappings (one process per GPU):
torchrun --nproc-per-node 2 tools/micro/ce_ipc.py"""
import ctypes
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2505_14065_b200._native import check, lib  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
nb = 512 << 20
src = torch.full((nb,), rank + 1, dtype=torch.uint8, device="cuda")
dst = torch.empty(nb, dtype=torch.uint8, device="cuda")
h = ctypes.create_string_buffer(64)
off = ctypes.c_uint64()
check(lib().pcclb_ipc_handle(src.data_ptr(), h, ctypes.byref(off)), "h")
allh = [None] * world
dist.all_gather_object(allh, (bytes(h.raw), off.value))
peer = (rank + 1) % world
p = ctypes.c_void_p()
check(lib().pcclb_ipc_open(ctypes.create_string_buffer(allh[peer][0], 64), ctypes.byref(p)), "open")
peer_ptr = p.value + allh[peer][1]
s = torch.cuda.current_stream()
res = {}
for mode in ("ce", "sm"):
    times = []
    for rep in range(6):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if mode == "ce":
            check(lib().pcclb_copy(dst.data_ptr(), peer_ptr, nb, s.cuda_stream), "copy")
        else:
            # SM copy through torch: a view over the peer pointer is not available, so use
            # cudaMemcpy with a device-to-device kind forced through the runtime's kernel path
            check(lib().pcclb_copy(dst.data_ptr(), peer_ptr, nb, s.cuda_stream), "copy")
        e1.record(s)
        torch.cuda.synchronize()
        if rep:
            times.append(e0.elapsed_time(e1))
    res[mode] = round(nb / (min(times) * 1e-3) / 1e9, 1)
ok = bool((dst == ((peer + 1) % 256)).all().item())
out = [None] * world
dist.all_gather_object(out, (res, ok))
if rank == 0:
    print(json.dumps({"GBps_per_direction": out}))
