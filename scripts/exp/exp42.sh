#!/bin/bash
# Pipelined compact kernel v2 (every prefetch as cp.async into shared memory,
# offset+count as one 8-byte entry): chunked (pipe) vs round-robin (pipe_rr)
# tile assignment vs the per-CTA kernel (main); parity on pipe; ncu of pipe.
set -u
O=gpurun_out/exp42
mkdir -p $O
TLBM_LIB=build/variants/pipe/libtlbm.so timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity_full.py tests/test_gpu_slabs.py -m gpu -q -x > $O/pytest_pipe.txt 2>&1
tail -2 $O/pytest_pipe.txt
for r in 1 2; do
for lib in main pipe pipe_rr; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.9,1.0 --precisions f64,f32 --storages compact --steps 20 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
for lib in pipe pipe_rr; do
for pr in f64; do
  TLBM_LIB=build/variants/$lib/libtlbm.so ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_${lib}_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages compact --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page details > $O/prof_${lib}_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page source --csv > $O/prof_${lib}_${pr}_p02_source.csv 2>&1
  rm -f $O/prof_${lib}_${pr}_p02.ncu-rep
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp42/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
