#!/bin/bash
# Development: build the product library with extra nvcc defines into
# variants/<name>/libmlck_b200.so (git-ignored, travels with gpurun; load it
# with MLCK_B200_LIB=variants/<name>/libmlck_b200.so).
#   scripts/build_variant.sh minb8 -DMLCK_REPLAY_MINB=8
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
out=$ROOT/variants/$name
mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-O3 -Xptxas -v $*"
for f in kernels capi log engine; do
  nvcc $FL -c $ROOT/paper_2412_15411_b200/csrc/$f.cu -o $out/$f.o 2> $out/$f.ptxas.log &
done
wait
nvcc $ARCH -shared -o $out/libmlck_b200.so $out/kernels.o $out/capi.o $out/log.o $out/engine.o -lcudart
