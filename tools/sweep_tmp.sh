source <(sed -n '/^run() {/,/^}/p' tools/qstep_sweep.sh)
ELEMS=1200000000; port=29650
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; echo tests=$?; tail -1 gpurun_out/t4.log
N=2 run PCCLB_QSTEP=1
N=4 run PCCLB_QSTEP=1
N=4 run PCCLB_GLAG=8
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 --workload quant > gpurun_out/b4_quant.json 2> gpurun_out/b4_quant.err; echo bench=$?; cat gpurun_out/b4_quant.json
