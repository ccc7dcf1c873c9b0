#!/bin/bash
# Stores of the compact kernels as IMAD.WIDE.U32 from one per-node base (no
# sign-extended LEA pairs): compact/nodes parity, slabs, ladder; sweep.
set -u
O=gpurun_out/exp49
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_compact.py tests/test_gpu_slabs.py tests/test_gpu_ladder.py -m gpu -q -x > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
for r in 1 2; do
  timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.7,1.0 --precisions f64,f32 --storages nodes,compact --steps 30 > $O/sweep_$r.jsonl 2>$O/sweep_$r.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp49/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
