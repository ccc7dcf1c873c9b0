#!/bin/bash
# Build an experimental libtlbm.so with extra -D flags on the step kernels:
#   scripts/build_variant.sh NAME "-DTLBM_MINB=12 -DTLBM_PULL_MODE=2"
# -> build/variants/NAME/libtlbm.so (select it with TLBM_LIB=...; used by
# scripts/step_sweep.py tuning runs).  The main objects come from `make`.
set -eu
NAME=$1; FLAGS=${2:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/variants/$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
NV="nvcc -O3 -std=c++20 $ARCH -lineinfo -fmad=false -Xptxas -v -Xcompiler -fPIC -I$ROOT/include --expt-relaxed-constexpr $FLAGS"
C=$ROOT/paper_1611_02445_b200/csrc
$NV -c -o $OUT/step_f32.o $C/step_f32.cu 2> $OUT/f32.log &
$NV -c -o $OUT/step_f64.o $C/step_f64.cu 2> $OUT/f64.log &
wait
O=$ROOT/paper_1611_02445_b200/lib/obj
nvcc $ARCH -shared -o $OUT/libtlbm.so $(ls $O/*.o | grep -v -E "step_f(32|64).o") \
    $OUT/step_f32.o $OUT/step_f64.o
echo $OUT/libtlbm.so
