"""Microbenchmark of the simplehash kernel variants (PCCLB_HASH_VARIANT).

Run one variant per process:  PCCLB_HASH_VARIANT=k python tools/hash_variants.py
Prints one JSON line: config-4 layout (whole, its two 1.05 GB entries alone,
the other 289 alone), a single 1.05 GB entry, and 64 equal 64 MiB entries
(HBM-bound case), each as ms and GB/s (CUDA events)."""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import llama3_8b_layout  # noqa: E402
from paper_2505_14065_b200.sharedstate import simplehash_many_async  # noqa: E402


def timeit(views, reps=5):
    """Per-call CUDA-event times; reports the median and the min."""
    import time

    out = torch.empty(len(views), dtype=torch.int64, device="cuda")
    simplehash_many_async(views, out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    host = []
    ev[0].record()
    for i in range(reps):
        t0 = time.perf_counter()
        simplehash_many_async(views, out)
        host.append((time.perf_counter() - t0) * 1e3)
        ev[i + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    ms = ts[len(ts) // 2]
    nb = sum(v.numel() * v.element_size() for v in views)
    return {"ms": round(ms, 3), "GBps": round(nb / ms / 1e6, 1), "min_ms": round(ts[0], 3),
            "max_ms": round(ts[-1], 3), "host_ms": round(max(host), 3)}, out.cpu().tolist()


layout = llama3_8b_layout()
total = sum(n for _, n in layout)
state = torch.empty(total, dtype=torch.bfloat16, device="cuda")
state.view(torch.int16).random_(-32768, 32767)
views, off = [], 0
for _, n in layout:
    views.append(state[off : off + n])
    off += n
res = {"variant": int(os.environ.get("PCCLB_HASH_VARIANT", "0"))}
res["config4"], digests = timeit(views, 7)
# the two largest entries (the bitsliced kernel's share) and the rest alone
res["config4_big2"], _ = timeit([views[0], views[-1]], 5)
res["config4_rest"], _ = timeit(views[1:-1], 5)
res["single_1GB"], _ = timeit([views[0]], 5)
eq = state[: 64 * (32 << 20)].view(64, -1)
res["64x64MiB"], _ = timeit([eq[i] for i in range(64)], 7)
if os.environ.get("HASH_SINGLE_16G"):  # config 4's single-entry stress case (the whole state as one entry)
    res["single_16GB"], _ = timeit([state.view(torch.uint8)], 3)
res["digest0"] = digests[0] & 0xFFFFFFFFFFFFFFFF
print(json.dumps(res), flush=True)
try:
    import pynvml

    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    print(json.dumps({"sm_mhz_after": pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                      "reasons": int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hd))}))
except Exception as exc:  # noqa: BLE001
    print(json.dumps({"nvml": str(exc)}))
