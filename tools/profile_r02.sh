#!/bin/bash
# Round-2 one-GPU ncu evidence (run under gpurun from the repo root). Every
# profiled command first runs plainly and must exit 0 (B200_PROFILING.md).
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
HASH="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity"
$HASH > $OUT/plain_hash.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_hash.csv $HASH > $OUT/ncu_launch_hash.log 2>&1
$HASH > $OUT/plain_hash2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"simplehash_(batch|big)" -s 4 -c 2 -o $OUT/prof_hash $HASH > $OUT/ncu_full_hash.log 2>&1
python tools/micro/hash_trace.py tools/micro/libs/trace.so > $OUT/trace.log 2>&1
CRC="python tools/crc_once.py"
$CRC > $OUT/plain_crc.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:crc32_seg -s 1 -c 1 -o $OUT/prof_crc $CRC > $OUT/ncu_full_crc.log 2>&1
echo done
