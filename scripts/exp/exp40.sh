#!/bin/bash
# Persistent software-pipelined compact kernel (TLBM_COMPACT_PIPE=1, cp.async
# staging two tiles ahead) vs the one-tile-group-per-CTA compact kernel:
# parity (compact tests on the variant), porosity sweep A/B on one box,
# ncu of both at porosity 0.2 (fp64, fp32).
set -u
O=gpurun_out/exp40
mkdir -p $O
V=build/variants/pipe/libtlbm.so
TLBM_LIB=$V timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity_full.py -m gpu -q -x > $O/pytest_pipe.txt 2>&1
tail -2 $O/pytest_pipe.txt
for r in 1 2; do
for lib in main pipe; do
  if [ $lib = main ]; then L=""; else L=$V; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.9,1.0 --precisions f64,f32 --storages compact --steps 20 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
for lib in main pipe; do
  if [ $lib = main ]; then L=""; else L=$V; fi
  for pr in f64 f32; do
  TLBM_LIB=$L ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_${lib}_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages compact --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page details > $O/prof_${lib}_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_${lib}_${pr}_p02.ncu-rep --page raw --csv > $O/prof_${lib}_${pr}_p02_raw.csv 2>&1
  rm -f $O/prof_${lib}_${pr}_p02.ncu-rep
  done
done
for pr in f64 f32; do
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_blocks_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages blocks --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_blocks_${pr}_p02.ncu-rep --page details > $O/prof_blocks_${pr}_p02_details.txt 2>&1
  rm -f $O/prof_blocks_${pr}_p02.ncu-rep
done
head -50 $O/sweep_*.jsonl
du -sh $O
