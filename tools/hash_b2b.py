import os, sys, torch
sys.path.insert(0, os.getcwd())
from bench import llama3_8b_layout
from paper_2505_14065_b200.sharedstate import simplehash_many_async
layout = llama3_8b_layout()
state = torch.empty(sum(n for _, n in layout), dtype=torch.bfloat16, device="cuda")
state.view(torch.int16).random_(-32768, 32767)
views, off = [], 0
for _, n in layout:
    views.append(state[off:off+n]); off += n
out = torch.empty(len(views), dtype=torch.int64, device="cuda")
for _ in range(3): simplehash_many_async(views, out)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
ev[0].record()
for i in range(20):
    simplehash_many_async(views, out); ev[i+1].record()
torch.cuda.synchronize()
ts = [ev[i].elapsed_time(ev[i+1]) for i in range(20)]
print("per-call:", [round(t,3) for t in ts], "avg", round(sum(ts)/20,3))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20): simplehash_many_async(views, out)
e1.record(); torch.cuda.synchronize()
print("b2b avg", round(e0.elapsed_time(e1)/20, 3))
