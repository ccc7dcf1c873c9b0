#!/bin/bash
# MRT (reference arithmetic) at 20 warps/SM (mw20) vs 16 (main) on the
# compact kernels: node-parallel and tile-parallel, packs p0.2 / p0.5 / 1.0.
set -u
for r in 1 2; do
for lib in main mw20; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for p in 0.2 0.5 1.0; do
  for tr in nodes tile; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity $p --variants mrt --steps 30 --storage compact --traversal $tr | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'p$p', '$tr', d['ms'], d['frac'])"
  done; done
done; done
