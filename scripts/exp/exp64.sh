#!/bin/bash
# fp32 MRT occupancy: 32 warps/SM (main) vs 40 (fw40) vs 24 (fw24); channel
# 256^3 blocks and the porosity-0.2 pack node-parallel.
set -u
for r in 1 2; do
for lib in main fw40 fw24; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel', d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --precision f32 --variants mrt --steps 50 --storage compact --traversal nodes | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'pack0.2 nodes', d['ms'], d['frac'])"
done; done
