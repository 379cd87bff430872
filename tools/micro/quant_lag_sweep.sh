# lag / slot knobs of the fused quantized schedule at W=2 (1.2 B f32)
run() { timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 tools/ring_phases.py 1200000000 quant 2>/dev/null | tail -1 | cut -c50-400; }
for e in "X=1" "PCCLB_GLAG=2" "PCCLB_GLAG=8" "PCCLB_GLAG=16" "PCCLB_QLAG=1" "PCCLB_QLAG=4" "PCCLB_QSLOTS=1"; do export $e; echo "$e: $(run)"; unset ${e%%=*}; done
