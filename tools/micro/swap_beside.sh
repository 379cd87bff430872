for f in tools/micro/libs/*.so; do
  cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so
  cp $f paper_2505_14065_b200/_lib/libpcclb200.so
  for b in 1 2 3; do echo "$f beside=$b: $(PCCLB_HASH_BESIDE=$b timeout 200 python tools/hash_variants.py 2>&1 | tail -2 | head -1)"; done
  cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so
done
