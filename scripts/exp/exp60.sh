#!/bin/bash
# fp64 block-store step, tiles per CTA: 2 (main) vs 1 vs 4 -- LBGK and MRT
# (reference and FMA arithmetic), channel 256^3.
set -u
O=gpurun_out/exp60
mkdir -p $O
for r in 1 2; do
for lib in main tpc1 tpc4; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for ar in reference fma; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f64 --arith $ar --variants full,mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$ar', d['variant'], d['ms'], d['frac'])"
  done
done; done
