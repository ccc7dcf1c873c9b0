#!/bin/bash
# LBGK: status word computed before the relaxation (lbst,
# TLBM_LBGK_STATUS_FIRST 1) vs after (main); same operations, different
# ptxas schedule.  256^3 channel (block store) and the porosity-0.2 pack
# (node-parallel), fp64 and fp32.
set -u
mkdir -p gpurun_out/exp76
for r in 1 2 3; do
for lib in main lbst; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for pr in f64 f32; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $pr --variants full --steps 100 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$pr channel', d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --precision $pr --variants full --steps 100 --storage compact --traversal nodes | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$pr pack0.2 nodes', d['ms'], d['frac'])"
  done
done; done 2>&1 | tee gpurun_out/exp76/ab.txt
