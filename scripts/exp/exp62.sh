#!/bin/bash
# fp64 MRT at one tile per CTA: occupancy 16/24 warps (main: reference/FMA)
# vs 20/28 (mw20) vs 12/20 (mw12).
set -u
for r in 1 2; do
for lib in main mw18 mw20 mw24; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for ar in reference; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f64 --arith $ar --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$ar', d['variant'], d['ms'], d['frac'])"
  done
done; done
