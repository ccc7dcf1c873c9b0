#!/bin/bash
# Build an experimental libtlbm.so with extra -D flags on the step kernels:
#   [ONLY=f32|f64] [SRC=dir] scripts/build_variant.sh NAME "-DTLBM_MINB=12 -DTLBM_PULL_MODE=2"
# -> build/variants/NAME/libtlbm.so (select it with TLBM_LIB=...; used by
# scripts/step_sweep.py tuning runs).  The main objects come from `make`.
set -eu
NAME=$1; FLAGS=${2:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/variants/$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
NV="nvcc -O3 -std=c++20 $ARCH -lineinfo -fmad=false -Xptxas -v -Xcompiler -fPIC -I$ROOT/include --expt-relaxed-constexpr $FLAGS"
# SRC=<dir> compiles the step units from a modified copy of csrc/ (an
# experiment that should not touch the tracked kernel sources)
C=${SRC:-$ROOT/paper_1611_02445_b200/csrc}
# ONLY=f32 / ONLY=f64 rebuilds one dtype and links the main build's other one
O=$ROOT/paper_1611_02445_b200/lib/obj
for d in f32 f64; do
  if [ -z "${ONLY:-}" ] || [ "${ONLY:-}" = $d ]; then
    $NV -c -o $OUT/step_$d.o $C/step_$d.cu 2> $OUT/$d.log &
  else
    cp $O/step_$d.o $OUT/step_$d.o
  fi
done
wait
nvcc $ARCH -shared -o $OUT/libtlbm.so $(ls $O/*.o | grep -v -E "step_f(32|64).o") \
    $OUT/step_f32.o $OUT/step_f64.o
echo $OUT/libtlbm.so
