# ncu (clocks unlocked) of ipc_qfinal_kernel with PCCLB_QDEBUG=$QDBG (default 29:
# A' alone, codes pushed locally, no tokens, no waits) next to the rmw2 micro's
# direct<2> kernel (3 CTAs/SM, 256 Ki items)
cd /root/repo
mkdir -p gpurun_out/qf9
export PCCLB_QDEBUG=${QDBG:-29}
timeout 600 ncu --clock-control none --target-processes all --set full --import-source on -k regex:ipc_qfinal -c 1 -o gpurun_out/qf9/qf${PCCLB_QDEBUG}_nc -f \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29583 tools/ring_phases.py 1200000000 quant > gpurun_out/qf9/log 2>&1
echo rc=$?
unset PCCLB_QDEBUG
timeout 300 ncu --clock-control none --set full --import-source on -k regex:direct -s 2 -c 1 -o gpurun_out/qf9/micro_direct_nc -f env ONLY=1 ./tools/micro/rmw2 > gpurun_out/qf9/micro.log 2>&1; echo rc=$?
