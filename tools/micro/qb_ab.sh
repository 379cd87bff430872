#!/bin/bash
# A/B of the fused quantized schedule's ready-flag block size (PCCLB_QB builds in tools/micro/libs)
cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/def.so
for rep in 1 2; do
for f in /tmp/def.so tools/micro/libs/*.so; do
  cp $f paper_2505_14065_b200/_lib/libpcclb200.so
  for N in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2986$N bench.py --gpus $N --workload quant > gpurun_out/qb.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/qb.json')); print('$f', $N, d['ms_per_step'], d['roofline']['frac'])"
  done
done; done
for f in tools/micro/libs/*.so; do cp $f paper_2505_14065_b200/_lib/libpcclb200.so; echo "$f: $(timeout 600 python -m pytest tests/test_ring_ipc_gpu.py tests/test_communicator_gpu.py -x -q 2>&1 | tail -1)"; done
cp /tmp/def.so paper_2505_14065_b200/_lib/libpcclb200.so
