#!/bin/bash
# Node-parallel step v3 (IMAD.WIDE addressing, own rank stored at bounce-back
# positions: no rank select) vs v3 + persistent cp.async record prefetch (npf).
set -u
O=gpurun_out/exp45
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_compact.py -m gpu -q -x > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
TLBM_LIB=build/variants/npf/libtlbm.so timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_slabs.py -m gpu -q -x -k "nodes or compact" > $O/pytest_npf.txt 2>&1
tail -2 $O/pytest_npf.txt
for r in 1 2; do
for lib in main npf; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.3,0.5,0.7,0.9,1.0 --precisions f64,f32 --storages nodes --steps 20 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
for lib in main npf; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
for pr in f64 f32; do
  TLBM_LIB=$L ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_${lib}_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages nodes --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page details > $O/prof_${lib}_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page raw --csv > $O/prof_${lib}_${pr}_p02_raw.csv 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page source --csv > $O/prof_${lib}_${pr}_p02_source.csv 2>&1
  rm -f $O/prof_${lib}_${pr}_p02.ncu-rep
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp45/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
