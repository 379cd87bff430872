"""One config-3-shaped quantized all-reduce of 8 logical peers on one GPU
(per-peer 150 M f32 = the W=8 chunk size times 1), for ncu captures of the
fused quantize->dequantize->accumulate hop kernel."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14065_b200 import LocalRing  # noqa: E402

w, n = 8, 150_000_000
g = torch.Generator(device="cuda").manual_seed(0)
bufs = [torch.randn(n, generator=g, device="cuda") * 1e-2 for _ in range(w)]
ring = LocalRing(w, backup=False)
for _ in range(2):
    assert ring.launch(bufs, "avg", quantize=True) == 0
torch.cuda.synchronize()
print("ok")
