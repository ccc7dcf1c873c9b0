#!/bin/bash
# fp32 MRT row sums in pairs (TLBM_MRT_PACKED 2: FFMA2(c, d, -0) products +
# FADD2 row sums) vs packed products only (pk1, round-2 main) and the paired
# form at 32/24 warps per SM (pk2w32); MRT parity tests on the main build.
set -u
mkdir -p gpurun_out/exp71
timeout 900 python -m pytest tests -m gpu -q -x -k "mrt or MRT" > gpurun_out/exp71/pytest_mrt.txt 2>&1; tail -1 gpurun_out/exp71/pytest_mrt.txt
for r in 1 2; do
for lib in main pk1 pk2w32; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel', d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --precision f32 --variants mrt --steps 50 --storage compact --traversal nodes | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'pack0.2 nodes', d['ms'], d['frac'])"
done; done 2>&1 | tee gpurun_out/exp71/ab.txt
