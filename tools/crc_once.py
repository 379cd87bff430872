"""CRC-32 of the config-4 state (291 entries, 16.06 GB) -- for ncu and timing."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import llama3_8b_layout  # noqa: E402
from paper_2505_14065_b200 import crc32_many  # noqa: E402

layout = llama3_8b_layout()
state = torch.empty(sum(n for _, n in layout), dtype=torch.bfloat16, device="cuda")
state.view(torch.int16).random_(-32768, 32767)
views, off = [], 0
for _, n in layout:
    views.append(state[off: off + n])
    off += n
crc32_many(views)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    crc32_many(views)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"crc32 config4: {ms:.3f} ms, {state.numel() * 2 / ms / 1e6:.1f} GB/s")
