#!/bin/bash
# fp32 node-parallel step, two nodes per thread: both records loaded before
# either gather (rec1st) vs record+gather per node in turn (main).
set -u
O=gpurun_out/exp59
mkdir -p $O
TLBM_LIB=build/variants/rec1st/libtlbm.so timeout 900 python -m pytest tests/test_gpu_compact.py -m gpu -q -x -k "nodes or equals" > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
for lib in main rec1st; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.8 --precisions f32 --storages nodes --steps 30 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp59/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
