#!/bin/bash
# fp32 node-parallel LBGK step: nodes per thread / warps per SM.
# main = 2 nodes at 32 warps/SM; npt3 = 3 at 24; npt4 = 4 at 16;
# npt2w40 = 2 at 40 (spills).  Sphere packs p 0.2 / 0.5 and the full box.
set -u
mkdir -p gpurun_out/exp73
for r in 1 2; do
for lib in main npt3 npt4 npt2w40; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for por in 0.2 0.5 1.0; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity $por --precision f32 --variants full --steps 50 --storage compact --traversal nodes | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'pack$por nodes', d['ms'], d['frac'])"
  done
done; done 2>&1 | tee gpurun_out/exp73/ab.txt
