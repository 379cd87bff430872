#!/bin/bash
# tools/micro/build_ring_variant.sh NAME "-DKNOB=V ..." -> tools/micro/libs/NAME.so
# (ring_ipc.cu rebuilt with the knobs, every other object from the default build)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
C=$ROOT/paper_2505_14065_b200/csrc
O=$ROOT/paper_2505_14065_b200/_lib/obj
T=$(mktemp -d)
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -I$ROOT/include \
  -Xcompiler -fPIC,-fvisibility=hidden -cudart static --expt-relaxed-constexpr $2 -c $C/ring_ipc.cu -o $T/ring_ipc.o
nvcc $ARCH -shared -cudart static -Xcompiler -fPIC -o $ROOT/tools/micro/libs/$1.so \
  $O/capi.o $O/kernels.o $O/hash.o $O/crc.o $O/ring_local.o $T/ring_ipc.o -lpthread -ldl -lrt
rm -rf $T
