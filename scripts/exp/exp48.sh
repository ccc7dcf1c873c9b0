#!/bin/bash
# fp32 node-parallel step shapes: 48 warps / 128 threads (main) vs 56 warps
# (32 registers), 256- and 64-thread CTAs.
set -u
O=gpurun_out/exp48
mkdir -p $O
for r in 1 2; do
for lib in main nw56 nt256 nt64; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,1.0 --precisions f32 --storages nodes --steps 30 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp48/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
