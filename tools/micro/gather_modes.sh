# plain all-reduce gather engines, 1 GiB f32 AVG (tools/ring_phases.py), W = $W
W=${W:-2}
run() { timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29582 tools/ring_phases.py ${N:-268435456} 2>/dev/null | tail -1 | cut -c50-400; }
for g in ${MODES:-push ce il}; do export PCCLB_GATHER=$g; echo "$g: $(run)"; done
