cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so
for v in prof; do
cp tools/micro/libs/$v.so paper_2505_14065_b200/_lib/libpcclb200.so
echo "== $v"; timeout 200 python tools/hash_variants.py 2>&1 | grep phase1 | head -4
done
cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so
