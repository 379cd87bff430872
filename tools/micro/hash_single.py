"""Hash one 1.05 GB entry (the config-4 embedding shape) a few times; for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2505_14065_b200.sharedstate import simplehash_many_async  # noqa: E402

x = torch.empty(128256 * 4096, dtype=torch.bfloat16, device="cuda")
x.view(torch.int16).random_(-32768, 32767)
out = torch.empty(1, dtype=torch.int64, device="cuda")
for _ in range(int(os.environ.get("REPS", "2"))):
    simplehash_many_async([x], out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
simplehash_many_async([x], out)
b.record()
torch.cuda.synchronize()
print(os.environ.get("PCCLB_HASH_VARIANT", "0"), "single entry ms", a.elapsed_time(b), hex(out.item() & (2**64 - 1)))
