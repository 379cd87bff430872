# ncu of one single-entry (1.05 GB) simplehash launch; run only after the same command exited 0 without ncu
ncu --set full --clock-control none --import-source on -k regex:simplehash_batch -c 1 --launch-skip 2 \
  -f -o gpurun_out/hash_single python tools/micro/hash_single.py > gpurun_out/ncu_hash_single.log 2>&1
