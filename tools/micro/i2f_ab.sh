#!/bin/bash
# A/B: dequantize codes with the 2^23 magic-number conversion (default) vs I2F.U8 (PCCLB_CODE_I2F build)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/i2f_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/i2f_tests.log
cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/new.so
for rep in 1 2; do
for v in new i2f; do
  if [ $v = new ]; then cp /tmp/new.so paper_2505_14065_b200/_lib/libpcclb200.so; else cp tools/micro/libs/i2f.so paper_2505_14065_b200/_lib/libpcclb200.so; fi
  for N in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2985$N bench.py --gpus $N --workload quant > gpurun_out/ab_$v$N.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v$N.json')); print('$v', $N, d['ms_per_step'], d['value'], d['roofline']['frac'])"
  done
done; done
cp /tmp/new.so paper_2505_14065_b200/_lib/libpcclb200.so
