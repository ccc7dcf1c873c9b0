#!/bin/bash
# fp32 MRT block-store kernel with packed row sums: 32 warps/SM (main) vs 28
# and 36; pk1 = packed products only at 40 (round-2 main); the node-parallel
# step (packed products, PACK 1) must be back at pk1's time.
set -u
mkdir -p gpurun_out/exp72
timeout 900 python -m pytest tests -m gpu -q -x -k "mrt or MRT" > gpurun_out/exp72/pytest_mrt.txt 2>&1; tail -1 gpurun_out/exp72/pytest_mrt.txt
for r in 1 2; do
for lib in main pk1 pkw28 pkw36; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel', d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --precision f32 --variants mrt --steps 50 --storage compact --traversal nodes | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'pack0.2 nodes', d['ms'], d['frac'])"
done; done 2>&1 | tee gpurun_out/exp72/ab.txt
