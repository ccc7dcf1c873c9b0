#!/bin/bash
# Node-parallel step v4: addresses as IMAD.WIDE.U32 with run-time scales
# (FMA pipe instead of LEA pairs on the ALU pipe), entry read for every pull
# with only the final offset selected.
set -u
O=gpurun_out/exp46
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_compact.py -m gpu -q -x > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
  timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.3,0.5,0.7,0.9,1.0 --precisions f64,f32 --storages nodes --steps 20 > $O/sweep_$r.jsonl 2>$O/sweep_$r.err
done
for pr in f64 f32; do
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages nodes --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_${pr}_p02.ncu-rep --page details > $O/prof_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_${pr}_p02.ncu-rep --page raw --csv > $O/prof_${pr}_p02_raw.csv 2>&1
  ncu -i $O/prof_${pr}_p02.ncu-rep --page source --csv > $O/prof_${pr}_p02_source.csv 2>&1
  rm -f $O/prof_${pr}_p02.ncu-rep
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp46/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
