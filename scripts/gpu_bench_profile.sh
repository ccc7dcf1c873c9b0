#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list, one full
# ncu capture of the step kernel.  Outputs under gpurun_out/$TAG/.
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
tail -c 3000 $OUT/bench.err
cat $OUT/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep \
    > $OUT/ncu_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
    -o $OUT/prof_step python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-sweep \
    > $OUT/ncu_full_run.log 2>&1
ls -la $OUT
