#!/bin/bash
# tools/micro/build_variant.sh SRC NAME "-DKNOB=V ..." -> tools/micro/libs/NAME.so
# (csrc/SRC.cu rebuilt with the knobs, every other object from the default build)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
C=$ROOT/paper_2505_14065_b200/csrc
O=$ROOT/paper_2505_14065_b200/_lib/obj
T=$(mktemp -d)
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p $ROOT/tools/micro/libs
nvcc $ARCH -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -I$ROOT/include \
  -Xcompiler -fPIC,-fvisibility=hidden -cudart static --expt-relaxed-constexpr $3 -c $C/$1.cu -o $T/$1.o
objs=""
for o in capi kernels hash crc ring_local ring_ipc; do
  if [ $o = $1 ]; then objs="$objs $T/$o.o"; else objs="$objs $O/$o.o"; fi
done
nvcc $ARCH -shared -cudart static -Xcompiler -fPIC -o $ROOT/tools/micro/libs/$2.so $objs -lpthread -ldl -lrt
rm -rf $T
