#!/bin/bash
# Fused quantized-step experiments (run under gpurun --gpus N from the repo root):
# per-phase device times of the NVLink ring for env variants.
N=${N:-2}
ELEMS=${ELEMS:-1200000000}
port=29600
run() {
  port=$((port+1))
  echo "== $*"
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N} --master-addr 127.0.0.1 \
    --master-port $port tools/ring_phases.py $ELEMS quant 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['total_ms'], d['phase_ms_per_rank'][0])"
}
run PCCLB_QSTEP=0
run PCCLB_QSTEP=1
run PCCLB_QDEBUG=1
run PCCLB_QDEBUG=2
run PCCLB_QDEBUG=3
run PCCLB_QLAG=4

run PCCLB_QSLOTS=1
run PCCLB_QSLOTS=4
run PCCLB_QSLOTS=1 PCCLB_QDEBUG=3
if [ -n "$NCU" ]; then
  PCCLB_QDEBUG=3 NCU_ARGS="--set full --clock-control none --import-source on -k regex:qstep -s 2 -c 1 -o gpurun_out/prof_qstep" \
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29700 --no-python tools/rank0_ncu.sh tools/ring_phases.py $ELEMS quant > gpurun_out/ncu_qstep.log 2>&1
  echo ncu=$?
fi
