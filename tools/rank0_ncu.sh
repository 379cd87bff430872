#!/bin/bash
# torchrun --nproc-per-node N --no-python tools/rank0_ncu.sh <script> [args]: rank 0 runs
# under ncu (NCU_ARGS), the other ranks run plainly. Only for kernels that do
# not wait on peers inside the kernel (e.g. PCCLB_QDEBUG=3): ncu replays them.
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu $NCU_ARGS python "$@"
else
  exec python "$@"
fi
