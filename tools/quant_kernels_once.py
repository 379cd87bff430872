"""Config-3-sized single-GPU kernel seams (n_c = 300 M f32): range, quantize,
dequant-accumulate with fused range -- for ncu captures and HBM GB/s."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14065_b200.collective import QuantScratch, dequant_accumulate, quantize_chunk_async  # noqa: E402

n = 300_000_000
x = torch.randn(n, device="cuda") * 1e-2
acc = torch.randn(n, device="cuda") * 1e-2
codes = torch.empty(n, dtype=torch.uint8, device="cuda")
sc = QuantScratch("cuda")
nxt = torch.zeros(4, dtype=torch.int32, device="cuda")
for _ in range(2):
    quantize_chunk_async(x, codes, sc)
    dequant_accumulate("sum", acc, codes, sc.meta, nxt)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
quantize_chunk_async(x, codes, sc)
e[1].record()
dequant_accumulate("sum", acc, codes, sc.meta, nxt)
e[2].record()
torch.cuda.synchronize()
q_ms, d_ms = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
print(json.dumps({"range+quantize_ms": round(q_ms, 4), "range+quantize_GBps": round((4 * n + 4 * n + n) / q_ms / 1e6, 1),
                  "dequant_acc_ms": round(d_ms, 4), "dequant_acc_GBps": round((n + 8 * n) / d_ms / 1e6, 1)}))
