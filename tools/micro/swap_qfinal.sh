# qfinal variants at W=2 (phase times of tools/ring_phases.py): each library
# in tools/micro/libs and the default build, under every PCCLB_QDEBUG value in
# $DBGS (default "0 9": normal, A' alone = B' items skipped without waits)
run() { timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 tools/ring_phases.py 1200000000 quant 2>/dev/null | tail -1 | cut -c50-400; }
for f in tools/micro/libs/${1:-qf}*.so default; do
  if [ $f != default ]; then cp paper_2505_14065_b200/_lib/libpcclb200.so /tmp/orig.so; cp $f paper_2505_14065_b200/_lib/libpcclb200.so; fi
  for d in ${DBGS:-0 9}; do echo "$f dbg$d: $(PCCLB_QDEBUG=$d run)"; done
  if [ $f != default ]; then cp /tmp/orig.so paper_2505_14065_b200/_lib/libpcclb200.so; fi
done
