for w in async quant allreduce; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 --workload $w > gpurun_out/b4_$w.json 2> gpurun_out/b4_$w.err; echo bench_$w=$?; cat gpurun_out/b4_$w.json; tail -3 gpurun_out/b4_$w.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 --impl reference --workload quant > gpurun_out/b4_ref_quant.json 2>&1; cat gpurun_out/b4_ref_quant.json | tail -1
