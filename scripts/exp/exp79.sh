#!/bin/bash
# fp32 block-store step at two tiles per CTA (tpc2, TLBM_TPC_F32 2) vs one
# (main): LBGK and MRT on the 256^3 channel, alternating, 3 rounds.
set -u
mkdir -p gpurun_out/exp79
for r in 1 2 3; do
for lib in main tpc2; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants full,mrt --steps 100 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', d['variant'], d['ms'], d['frac'])"
done; done 2>&1 | tee gpurun_out/exp79/ab.txt
