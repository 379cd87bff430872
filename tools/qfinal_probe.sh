# phases of the quantized schedule at W=2 (1.2 B f32): default, lag variants, no-wait debug
for env in "X=1" "PCCLB_GLAG=2" "PCCLB_GLAG=8" "PCCLB_QDEBUG=1"; do
  echo "$env: $(env $env timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/ring_phases.py 1200000000 quant 2>/dev/null | tail -1 | cut -c1-400)"
done
