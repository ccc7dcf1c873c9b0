#!/bin/bash
# On the GPU box: one ncu --set full capture of the bench's step kernel per
# precision (the launch after 6 warm-up launches), exported as raw CSV for
# scripts/update_traffic.py.  Outputs under gpurun_out/$TAG/.
set -u
TAG=${1:-traffic}
O=gpurun_out/$TAG
mkdir -p $O
for p in f64 f32; do
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
      -o $O/prof_step_$p python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-sweep \
      --precision $p > /dev/null 2>&1
  ncu -i $O/prof_step_$p.ncu-rep --page raw --csv > $O/prof_step_${p}_raw.csv 2>&1
  ncu -i $O/prof_step_$p.ncu-rep --page details > $O/prof_step_${p}_details.txt 2>&1
done
