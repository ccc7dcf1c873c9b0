#!/bin/bash
# Node-parallel step: L2 prefetch of the node records one (l2pf1) or two
# (l2pf2) waves of resident CTAs ahead vs none (main).
set -u
O=gpurun_out/exp47
mkdir -p $O
TLBM_LIB=build/variants/l2pf1/libtlbm.so timeout 900 python -m pytest tests/test_gpu_compact.py -m gpu -q -x -k nodes > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
for lib in main l2pf1 l2pf2; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.9,1.0 --precisions f64,f32 --storages nodes --steps 20 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp47/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
