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
big = os.environ.get("BIG") == "1"  # 1 GiB tensors, each rank copies the half it "owns" (rank+1)%2
src_full = torch.full((2 * nb if big else nb,), rank + 1, dtype=torch.uint8, device="cuda")
if os.environ.get("RAND") == "1":  # incompressible contents
    src_full.random_(0, 256)
src = src_full
dst = torch.empty(nb, dtype=torch.uint8, device="cuda")
if os.environ.get("RAND") == "1":
    dst.random_(0, 256)
h = ctypes.create_string_buffer(64)
off = ctypes.c_uint64()
check(lib().pcclb_ipc_handle(src.data_ptr(), h, ctypes.byref(off)), "h")
allh = [None] * world
dist.all_gather_object(allh, (bytes(h.raw), off.value))
peer = (rank + 1) % world
p = ctypes.c_void_p()
check(lib().pcclb_ipc_open(ctypes.create_string_buffer(allh[peer][0], 64), ctypes.byref(p)), "open")
peer_ptr = p.value + allh[peer][1]
own_off = ((rank + 1) % 2) * nb if big else 0
peer_ptr += own_off
s = torch.cuda.current_stream()
res = {}
for mode in ("ce", "push", "ce1g", "push_after_write", "push_after_pull", "pull_then_push", "pull_sleep_push"):
    times = []
    for rep in range(6):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if mode == "ce":  # pull: local <- peer
            check(lib().pcclb_copy(dst.data_ptr(), peer_ptr, nb, s.cuda_stream), "copy")
        elif mode == "push":  # push: peer <- local (into the peer's src tensor: it is refilled below)
            check(lib().pcclb_copy(peer_ptr, src_full.data_ptr() + own_off, nb, s.cuda_stream), "copy")
        elif mode == "push_after_write":  # the source was just written by SMs (like the fold's result)
            e0 = torch.cuda.Event(enable_timing=True)
            dst.fill_(7)
            e0.record(s)
            check(lib().pcclb_copy(peer_ptr, dst.data_ptr(), nb, s.cuda_stream), "copy")
        elif mode == "push_after_pull":  # SM remote loads of the peer buffer first (like the fold)
            e0 = torch.cuda.Event(enable_timing=True)
            acc = dst.view(torch.float32)
            check(lib().pcclb_accumulate(acc.data_ptr(), peer_ptr, acc.numel(), 1, 1, s.cuda_stream), "acc")
            torch.cuda.synchronize()
            dist.barrier()
            e0.record(s)
            check(lib().pcclb_copy(peer_ptr, src_full.data_ptr() + own_off, nb, s.cuda_stream), "copy")
        elif mode in ("pull_then_push", "pull_sleep_push"):  # stream-ordered, no host sync in between
            e0 = torch.cuda.Event(enable_timing=True)
            acc = dst.view(torch.float32)
            check(lib().pcclb_accumulate(acc.data_ptr(), peer_ptr, acc.numel(), 1, 1, s.cuda_stream), "acc")
            if mode == "pull_sleep_push":
                torch.cuda._sleep(1_000_000)  # ~0.5 ms at 1.9 GHz
            e0.record(s)
            check(lib().pcclb_copy(peer_ptr, src_full.data_ptr() + own_off, nb, s.cuda_stream), "copy")
        else:  # two 512 MiB pulls back to back
            check(lib().pcclb_copy(dst.data_ptr(), peer_ptr, nb, s.cuda_stream), "copy")
            check(lib().pcclb_copy(dst.data_ptr(), peer_ptr, nb, s.cuda_stream), "copy")
        e1.record(s)
        torch.cuda.synchronize()
        if rep:
            times.append(e0.elapsed_time(e1))
    res[mode] = round(nb * (2 if mode == "ce1g" else 1) / (min(times) * 1e-3) / 1e9, 1)
    dist.barrier()
    if os.environ.get("RAND") == "1":
        src.random_(0, 256)
    else:
        src.fill_(rank + 1)
    torch.cuda.synchronize()
    dist.barrier()
ok = bool((dst == ((peer + 1) % 256)).all().item())
out = [None] * world
dist.all_gather_object(out, (res, ok))
if rank == 0:
    print(json.dumps({"GBps_per_direction": out}))
