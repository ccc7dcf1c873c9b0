#!/bin/bash
# MRT: committed order (main: deviations, then the status word) vs lazy0
# (status word first, then all deviations; otherwise the same operations)
set -u
mkdir -p gpurun_out/exp75
for r in 1 2; do
for lib in main lazy0; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for pr in f64 f32; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $pr --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$pr channel', d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --precision $pr --variants mrt --steps 50 --storage compact --traversal nodes | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$pr pack0.2 nodes', d['ms'], d['frac'])"
  done
done; done 2>&1 | tee gpurun_out/exp75/ab.txt
