#!/bin/bash
# W=8 on a 4-GPU box: two ranks per GPU (time-sliced contexts). Correctness of
# every ring scenario and a bench smoke run; timings mean nothing here.
mkdir -p gpurun_out/w8r2
timeout 900 python tests/mp_ring_worker.py 8 29611 gpurun_out/w8r2 golden faults registered qedge ext large_small > gpurun_out/w8r2.log 2>&1; echo ring_rc=$?
python - <<'P'
import json,glob
bad=0;tot=0
for f in sorted(glob.glob('gpurun_out/w8r2/rank*.json')):
    d=json.load(open(f)); tot+=len(d['checks']); b=[c for c in d['checks'] if not c['ok']]; bad+=len(b)
    if d['errors'] or b: print(f, d['errors'][:1], b[:3])
print('w8 checks', tot, 'failed', bad)
P
tail -3 gpurun_out/w8r2.log
for wl in allreduce quant; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 8 --steps 3 --warmup 3 --workload $wl --no-e2e > gpurun_out/w8r2_$wl.json 2> gpurun_out/w8r2_$wl.err; echo bench8_${wl}_rc=$?
python -c "import json; d=json.load(open('gpurun_out/w8r2_$wl.json')); print('$wl', d['value'], d['ms_per_step'], d['parity'])"
done
