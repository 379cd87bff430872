rm -rf /tmp/di && mkdir -p /tmp/di
python - <<'PY' &
import sys, time
sys.path.insert(0, "baseline/_ref")
from churncomm.master import MasterConfig, MasterServer
s = MasterServer("127.0.0.1", 29666, MasterConfig(pool_size=1, probe_bytes=64*1024, vote_timeout=15.0)).start()
time.sleep(120)
PY
sleep 3
python tests/dropin_worker.py 0 2 29666 29667 /tmp/di & p0=$!
python tests/dropin_worker.py 1 2 29666 29667 /tmp/di & p1=$!
wait $p0; wait $p1
for r in 0 1; do python -c "
import json; d=json.load(open('/tmp/di/rank$r.json')); print($r, d['checks']); print(''.join(d['errors'])[-2500:])"; done
