# qfinal variants at W=2 (phase times of tools/ring_phases.py)
for f in tools/micro/libs/qf*.so; do
  cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so
  cp $f paper_2505_14065_b200/_lib/libpcclb200.so
  echo "$f: $(timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 tools/ring_phases.py 1200000000 quant 2>/dev/null | tail -1 | cut -c50-260)"
  cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so
done
