#!/bin/bash
# Round-end validation as the driver runs it (fresh box): smoke, every GPU
# test, the default bench line and the reference arm.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final/smoke.log
python bench.py --impl reference > gpurun_out/final/ref_n1.json 2> gpurun_out/final/ref_n1.err; echo ref1=$?
python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err; echo bench1=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final/tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/final/tests.log
python - <<'P'
import json
for f in ["ref_n1", "bench_n1"]:
    d = json.load(open(f"gpurun_out/final/{f}.json"))
    print(f, d["value"], d["unit"], d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("parity") or {}).get("status"), (d.get("e2e") or {}).get("value"), d.get("clocks", {}).get("sm_mhz") if d.get("clocks") else None)
P
