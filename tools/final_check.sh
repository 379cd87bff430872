#!/bin/bash
# Round-end validation on a 4-GPU box: smoke, every GPU test, default bench lines.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; echo tests=$?; tail -1 gpurun_out/t4.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench1=$?
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2982$N bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench$N=$?
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2983$N bench.py --gpus $N --workload quant > gpurun_out/bench_q$N.json 2> gpurun_out/bench_q$N.err; echo benchq$N=$?
done
for f in gpurun_out/bench_n1.json gpurun_out/bench_n2.json gpurun_out/bench_n4.json gpurun_out/bench_q2.json gpurun_out/bench_q4.json; do
  python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['unit'], d['ms_per_step'], d['roofline'].get('frac'))"
done
