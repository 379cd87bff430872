#!/bin/bash
# run tools/hash_variants.py against alternative builds of the library
for f in tools/micro/libs/*.so; do
  cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so
  cp $f paper_2505_14065_b200/_lib/libpcclb200.so
  echo "$f: $(timeout 200 python tools/hash_variants.py 2>&1 | tail -2 | head -1)"
  cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so
done
echo "default: $(timeout 200 python tools/hash_variants.py 2>&1 | tail -2 | head -1)"
