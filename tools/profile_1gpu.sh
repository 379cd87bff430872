#!/bin/bash
# One-GPU ncu evidence (run under gpurun from the repo root). Every profiled
# command first runs plainly and must exit 0 (B200_PROFILING.md rules).
set -u
OUT=gpurun_out
HASH="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
LOCAL="python bench.py --workload local --steps 2 --warmup 3 --no-e2e"
QLOCAL="python tools/local_quant_once.py"
$HASH > $OUT/plain_hash.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_hash.csv $HASH > $OUT/ncu_launch_hash.log 2>&1
$HASH > $OUT/plain_hash2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:simplehash_batch -s 3 -c 1 -o $OUT/prof_hash $HASH > $OUT/ncu_full_hash.log 2>&1
$LOCAL > $OUT/plain_local.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:local_fold_all -s 3 -c 1 -o $OUT/prof_local_fold $LOCAL > $OUT/ncu_full_local.log 2>&1
$QLOCAL > $OUT/plain_qlocal.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:local_q_hop -s 2 -c 1 -o $OUT/prof_local_qhop $QLOCAL > $OUT/ncu_full_qlocal.log 2>&1
echo done
