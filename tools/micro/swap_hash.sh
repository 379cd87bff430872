#!/bin/bash
# config-4 hash timing (tools/hash_b2b.py) with each library in tools/micro/libs/${1}*.so and the default build
for f in tools/micro/libs/${1:-h}*.so default; do
  if [ $f != default ]; then cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so; cp $f paper_2505_14065_b200/_lib/libpcclb200.so; fi
  echo "$f: $(timeout 200 python tools/hash_b2b.py 2>&1 | tail -1) $(timeout 200 python tools/hash_b2b.py 2>&1 | tail -1)"
  if [ $f != default ]; then cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so; fi
done
