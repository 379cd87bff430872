#!/bin/bash
# W=8 on a 4-GPU box (two ranks per GPU): fault/registered/qedge/large scenarios, quantized + async benches.
mkdir -p gpurun_out/w8f
timeout 900 python tests/mp_ring_worker.py 8 29641 gpurun_out/w8f faults registered qedge large > gpurun_out/w8f.log 2>&1; echo scen_rc=$?
python - <<'P'
import json,glob
bad=0;tot=0
for f in sorted(glob.glob('gpurun_out/w8f/rank*.json')):
    d=json.load(open(f)); tot+=len(d['checks']); b=[c for c in d['checks'] if not c['ok']]; bad+=len(b)
    if d['errors'] or b: print(f, d['errors'][:1], b[:3])
print('w8 scenario checks', tot, 'failed', bad)
P
tail -3 gpurun_out/w8f.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 8 --steps 3 --warmup 3 --workload quant --elems 150000000 > gpurun_out/w8_q.json 2> gpurun_out/w8_q.err; echo benchq8_rc=$?
head -c 400 gpurun_out/w8_q.json; tail -3 gpurun_out/w8_q.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 8 --steps 3 --warmup 3 --workload async --elems 64000000 > gpurun_out/w8_a.json 2> gpurun_out/w8_a.err; echo bencha8_rc=$?
head -c 400 gpurun_out/w8_a.json; tail -3 gpurun_out/w8_a.err
