#!/bin/bash
# Development timing variants of the 2b = 32 pair solve: builds
# build/exp<k>/libsvdk.so with -DSVDK_PROBES -DSVDK_EXP=<k> (switches are added
# to csrc/jacobi.cu per experiment and removed after; k = 0 is production).
# Run on the GPU: for k in ...; do SVDK_LIB=build/exp$k/libsvdk.so python tools/eig_probe.py 1024; done
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_1906_12085_b200/csrc
make -C "$ROOT/paper_1906_12085_b200" -j >/dev/null
OBJS=$(ls "$ROOT"/build/svdk/*.o | grep -v '/jacobi.o$')
for k in "$@"; do
  mkdir -p "$ROOT/build/exp$k"
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -I"$ROOT/include" -I"$CSRC" --expt-relaxed-constexpr -DSVDK_PROBES -DSVDK_EXP=$k \
     -c "$CSRC/jacobi.cu" -o "$ROOT/build/exp$k/jacobi.o" &&
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$ROOT/build/exp$k/libsvdk.so" \
     $OBJS "$ROOT/build/exp$k/jacobi.o" -lnccl -lpthread -ldl -lrt) &
done
wait
