#!/bin/bash
# Is the block-store step on mid-porosity packs bound by DRAM traffic
# (sector over-fetch) or by idle lanes?  DRAM bytes and throughput (ncu) of
# the block-store and the node-parallel steps at porosity 0.5 / 0.7.
set -u
O=gpurun_out/exp69
mkdir -p $O
for p in 0.5 0.7; do for pr in f32 f64; do for st in blocks nodes; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none \
    -k regex:step_kernel -s 5 -c 1 --csv --log-file $O/ncu_${st}_${pr}_p$p.csv \
    python scripts/porosity_sweep.py --porosities $p --precisions $pr --storages $st --steps 3 --warmup 5 > $O/run_${st}_${pr}_p$p.jsonl 2>&1
done; done; done
for f in $O/ncu_*.csv; do echo "== $f"; grep -E "dram__|gpu__time|warps_active|thread_inst" $f | awk -F'","' '{print $13, $14, $15}'; done
