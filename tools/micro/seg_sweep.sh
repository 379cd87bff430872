cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so
for rep in 1 2; do
for f in tools/micro/libs/*.so default; do
  if [ $f != default ]; then cp $f paper_2505_14065_b200/_lib/libpcclb200.so; else cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so; fi
  echo "$f: $(timeout 200 python tools/hash_variants.py 2>&1 | tail -2 | head -1)"
done; done
for f in tools/micro/libs/*.so; do cp $f paper_2505_14065_b200/_lib/libpcclb200.so; echo "$f test: $(timeout 300 python -m pytest tests/test_hash_gpu.py -x -q 2>&1 | tail -1)"; done
cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so
