# qfinal isolation at W=2 (1.2 B f32): 8 = B' items skipped (A' only), 4 = A' pushes locally (no NVLink), 12 = both
for env in "X=1" "PCCLB_QDEBUG=8" "PCCLB_QDEBUG=4" "PCCLB_QDEBUG=12" "PCCLB_QDEBUG=9"; do
  echo "$env: $(env $env timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/ring_phases.py 1200000000 quant 2>/dev/null | tail -1 | cut -c50-400)"
done
