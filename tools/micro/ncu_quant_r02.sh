# ncu --set full (clocks unlocked) of the fused quantized kernels at W=2,
# config-3 shape; PCCLB_QDEBUG=1 (consumers never wait) so each replayed
# kernel is self-contained. Numbers under ncu are not bench values.
mkdir -p gpurun_out/r02q
export PCCLB_QDEBUG=1
timeout 900 ncu --clock-control none --target-processes all --set full --import-source on -k regex:"ipc_q(step|final)" -c 4 \
  -o gpurun_out/r02q/quant_w2 -f \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29583 tools/ring_phases.py 1200000000 quant > gpurun_out/r02q/log 2>&1
echo rc=$?
