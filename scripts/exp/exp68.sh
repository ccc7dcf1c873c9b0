#!/bin/bash
# fp64 node-parallel step CTA size: 128 threads (main) vs 64 vs 256.
set -u
O=gpurun_out/exp68
mkdir -p $O
for r in 1 2; do
for lib in main nt64 nt256; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.8 --precisions f64 --storages nodes --steps 30 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp68/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
