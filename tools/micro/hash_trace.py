"""Timeline of the config-4 hash launch from a PCCLB_HASH_TRACE build:
per-kernel CTA start/end (globaltimer) and how much the batch and big-entry
kernels actually share SMs. usage: python tools/micro/hash_trace.py lib.so"""

import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
lib_path = sys.argv[1]
import paper_2505_14065_b200._native as nat  # noqa: E402

nat.LIB_PATH = lib_path
from bench import llama3_8b_layout  # noqa: E402
from paper_2505_14065_b200.sharedstate import simplehash_many_async  # noqa: E402

lib = ctypes.CDLL(lib_path)
layout = llama3_8b_layout()
total = sum(n for _, n in layout)
state = torch.empty(total, dtype=torch.bfloat16, device="cuda")
state.view(torch.int16).random_(-32768, 32767)
views, off = [], 0
for _, n in layout:
    views.append(state[off : off + n])
    off += n
out = torch.empty(len(views), dtype=torch.int64, device="cuda")
buf = (ctypes.c_ulonglong * (8192 * 4))()
for _ in range(3):
    simplehash_many_async(views, out)
torch.cuda.synchronize()
lib.pcclb_debug_hash_trace(buf, 8192, 1)
simplehash_many_async(views, out)
torch.cuda.synchronize()
n = lib.pcclb_debug_hash_trace(buf, 8192, 1)
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4)[:n].astype(np.int64)
t0 = a[:, 2].min()
for kind, name in ((1, "batch"), (2, "big")):
    k = a[a[:, 0] == kind]
    if len(k) == 0:
        continue
    st, en = (k[:, 2] - t0) / 1e3, (k[:, 3] - t0) / 1e3
    print(f"{name}: {len(k)} CTAs on {len(set(k[:, 1]))} SMs; start {st.min():.0f}-{st.max():.0f} us, "
          f"end {en.min():.0f}-{en.max():.0f} us; starts>100us: {(st > 100).sum()}")
b, g = a[a[:, 0] == 1], a[a[:, 0] == 2]
shared = 0
for sm in set(g[:, 1]):
    gi = g[g[:, 1] == sm]
    bi = b[b[:, 1] == sm]
    for x in gi:
        for y in bi:
            if min(x[3], y[3]) > max(x[2], y[2]):
                shared += 1
print("big CTAs overlapping a batch CTA on the same SM:", shared)
it = a[a[:, 0] == 3]
if len(it):
    nb = it[:, 1] >> 16
    st, en = (it[:, 2] - t0) / 1e3, (it[:, 3] - t0) / 1e3
    print(f"items: {len(it)}")
    for size in sorted(set(nb.tolist()), reverse=True):
        m = nb == size
        d = en[m] - st[m]
        rate = size / 2 / (d * 1e-6) / 1e9  # one lane group = half the entry
        print(f"  entry {size / 1e6:8.1f} MB x{m.sum():4d}: start {st[m].min():6.0f}-{st[m].max():6.0f} us, "
              f"dur {d.min():6.0f}-{np.median(d):6.0f}-{d.max():6.0f} us, per-item {np.median(rate):5.1f} GB/s, "
              f"end max {en[m].max():6.0f}")
    late = np.argsort(-en)[:12]
    print("  last items (MB, start, end, sm):", [(round(nb[i] / 1e6, 1), round(st[i]), round(en[i]), int(it[i, 1] & 0xffff)) for i in late])
