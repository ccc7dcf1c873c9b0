#!/bin/bash
# exp40 again with the 16-byte-aligned stage (pipe kernel), plus the TMA
# read/write-only probe (scripts/probes/tma_probe.cu).
set -u
O=gpurun_out/exp41
mkdir -p $O
./scripts/probes/tma_probe > $O/tma_probe.jsonl 2>&1
cat $O/tma_probe.jsonl
V=build/variants/pipe/libtlbm.so
TLBM_LIB=$V timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity_full.py -m gpu -q -x > $O/pytest_pipe.txt 2>&1
tail -2 $O/pytest_pipe.txt
for r in 1 2; do
for lib in main pipe; do
  if [ $lib = main ]; then L=""; else L=$V; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.9,1.0 --precisions f64,f32 --storages compact --steps 20 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
for pr in f64 f32; do
  TLBM_LIB=$V ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_pipe_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages compact --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_pipe_${pr}_p02.ncu-rep --page details > $O/prof_pipe_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_pipe_${pr}_p02.ncu-rep --page raw --csv > $O/prof_pipe_${pr}_p02_raw.csv 2>&1
  ncu -i $O/prof_pipe_${pr}_p02.ncu-rep --page source --csv > $O/prof_pipe_${pr}_p02_source.csv 2>&1
  rm -f $O/prof_pipe_${pr}_p02.ncu-rep
done
ncu --set full --clock-control none -k regex:bulk_rw -c 1 -o $O/prof_bulk ./scripts/probes/tma_probe 262144 2 > /dev/null 2>&1
ncu -i $O/prof_bulk.ncu-rep --page details > $O/prof_bulk_details.txt 2>&1; rm -f $O/prof_bulk.ncu-rep
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp41/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['ms_per_step'], round(d['bu'],4))
PY
du -sh $O
