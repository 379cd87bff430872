"""Stress the fused quantized schedule against the barrier-per-step schedule:
K seeded ops, both engines on copies of the same input, outputs must be
bit-identical on every rank (a flag/ordering race would show as a mismatch).
torchrun --nproc-per-node N tools/qstress.py [K] [elems]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_14065_b200.ring_ipc import DeviceRing, init_from_env  # noqa: E402

rank, world, local = init_from_env("gloo")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_003
dev = torch.device("cuda", local)
fused = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, True), slots=2)
barr = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, True), slots=16)
bad = 0
ops = ["avg", "sum", "max", "min"]
for i in range(K):
    g = torch.Generator(device=dev).manual_seed(1000 * i + rank)
    x = torch.randn(n, generator=g, device=dev) * (10.0 ** (i % 5 - 2))
    a, b = x.clone(), x.clone()
    op = ops[i % 4]
    fused.run_all_reduce(a, op, quantize=True)
    barr.run_all_reduce(b, op, quantize=True)
    if not torch.equal(a.view(torch.int32), b.view(torch.int32)):
        bad += 1
got = [None] * world
torch.distributed.all_gather_object(got, bad)
if rank == 0:
    print(json.dumps({"world": world, "ops": K, "elems": n, "mismatching_ops_per_rank": got}))
fused.close()
barr.close()

# two fused engines running at once on two streams (the communicator's two
# slots): results must equal the sequential barrier-schedule results
e0 = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, True), slots=2)
e1 = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, True), slots=2)
barr = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, 4, True), slots=16)
s0, s1 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
bad2 = 0
for i in range(K // 2):
    g = torch.Generator(device=dev).manual_seed(7000 + 1000 * i + rank)
    x0 = torch.randn(n, generator=g, device=dev)
    x1 = torch.randn(n, generator=g, device=dev) * 3
    a0, a1, b0, b1 = x0.clone(), x1.clone(), x0.clone(), x1.clone()
    torch.cuda.synchronize(dev)
    t0 = e0.all_reduce_async(a0, "avg", quantize=True, stream=s0)
    t1 = e1.all_reduce_async(a1, "avg", quantize=True, stream=s1)
    e0.await_reduce(t0)
    e1.await_reduce(t1)
    barr.run_all_reduce(b0, "avg", quantize=True)
    barr.run_all_reduce(b1, "avg", quantize=True)
    bad2 += int(not torch.equal(a0.view(torch.int32), b0.view(torch.int32)))
    bad2 += int(not torch.equal(a1.view(torch.int32), b1.view(torch.int32)))
got = [None] * world
torch.distributed.all_gather_object(got, bad2)
if rank == 0:
    print(json.dumps({"concurrent_pairs": K // 2, "mismatching_ops_per_rank": got}))
