#!/bin/bash
# MRT deviations on demand (TLBM_MRT_LAZY 1, main) vs all 19 up front
# (lazy0); with the lazy form, fp64 MRT at 24 / 28 warps per SM and fp32
# block-store MRT at 40 (lz24), fp32 compact MRT at 40 (lz28).
set -u
mkdir -p gpurun_out/exp74
timeout 900 python -m pytest tests -m gpu -q -x -k "mrt or MRT" > gpurun_out/exp74/pytest_mrt.txt 2>&1; tail -1 gpurun_out/exp74/pytest_mrt.txt
for r in 1 2; do
for lib in main lazy0 lz24 lz28; do
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
done; done 2>&1 | tee gpurun_out/exp74/ab.txt
