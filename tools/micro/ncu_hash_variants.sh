# one ncu invocation over both variants (children followed)
ncu --set full --clock-control none --import-source on -k regex:simplehash_batch -c 2 --launch-skip 2 \
  --target-processes all -f -o gpurun_out/hash_v01 bash -c 'PCCLB_HASH_VARIANT=0 REPS=2 python tools/micro/hash_single.py; PCCLB_HASH_VARIANT=1 REPS=2 python tools/micro/hash_single.py' > gpurun_out/ncu_hash_v01.log 2>&1
