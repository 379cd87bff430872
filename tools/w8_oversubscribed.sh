#!/bin/bash
# W=8 dry run on a 4-GPU box: two ranks per GPU (time-sliced contexts), golden ring cases + a short bench.
nvidia-smi -L
mkdir -p gpurun_out/w8
timeout 600 python tests/mp_ring_worker.py 8 29611 gpurun_out/w8 golden > gpurun_out/w8_golden.log 2>&1; echo golden_rc=$?
python - <<'P'
import json,glob
bad=0;tot=0
for f in sorted(glob.glob('gpurun_out/w8/rank*.json')):
    d=json.load(open(f)); tot+=len(d['checks']); b=[c for c in d['checks'] if not c['ok']]; bad+=len(b)
    if d['errors'] or b: print(f, d['errors'][:1], b[:3])
print('w8 checks', tot, 'failed', bad)
P
tail -5 gpurun_out/w8_golden.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 8 --steps 3 --warmup 3 > gpurun_out/w8_bench.json 2> gpurun_out/w8_bench.err; echo bench8_rc=$?
cat gpurun_out/w8_bench.json; tail -5 gpurun_out/w8_bench.err
