# per-phase device times of the small path and the multi-kernel path at W=2
for n in 262144 1048576 4194304; do
  for sm in 8388608 0; do
    PCCLB_SMALL_MAX=$sm timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 tools/ring_phases.py $n 2>/dev/null | tail -1 | cut -c1-300
  done
done
