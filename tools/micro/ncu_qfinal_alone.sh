# ncu --set full of ipc_qfinal_kernel alone (PCCLB_QDEBUG=9: B' items skipped,
# no waits, so the replayed kernel is self-contained), W=2, config-3 shape
mkdir -p gpurun_out/qf9
export PCCLB_QDEBUG=${QDBG:-9}
timeout 600 ncu --target-processes all --set full --import-source on -k regex:${KNAME:-ipc_qfinal} -c 1 -o gpurun_out/qf9/${OUT:-qf9} -f \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29583 tools/ring_phases.py 1200000000 quant > gpurun_out/qf9/log 2>&1
echo rc=$?
tail -3 gpurun_out/qf9/log
