# timing sweep (median / min / max of 7 calls), two passes
for v in 0 1 2 3; do PCCLB_HASH_VARIANT=$v timeout 300 python -m pytest tests/test_hash_gpu.py -x -q 2>&1 | tail -1; done
for rep in 1 2; do
for v in 0 1 2 3; do echo "v=$v $(PCCLB_HASH_VARIANT=$v timeout 200 python tools/hash_variants.py 2>&1 | tail -1)"; done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
