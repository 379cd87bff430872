for k in death_plain death_quant death_plain; do
  rm -rf /tmp/dd && mkdir -p /tmp/dd
  timeout 300 python tests/mp_ring_worker.py 3 29577 /tmp/dd $k > /dev/null 2>gpurun_out/death_$k.err; echo "$k rc=$?"
  python -c "
import json
for r in range(2):
    d=json.load(open('/tmp/dd/rank%d.json'%r)); print(r, [(c['name'], c['ok']) for c in d['checks']], d['errors'][:1])"
done
