# sweep with the small path forced on (1 GiB cap) and off, W=2 and W=4
for W in 2 4; do
  for sm in 0 1073741824; do
    PCCLB_SMALL_MAX=$sm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2960$W bench.py --gpus $W --workload sweep > gpurun_out/sw_${W}_$sm.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/sw_${W}_$sm.json'))
print('W=$W small_max=$sm', [(r['bytes']>>20, r['us_per_op']) for r in d['config']['sweep']])"
  done
done
