#!/bin/bash
# Copy the summaries of a final evidence pass (scripts/exp/r2c_final.sh TAG)
# from gpurun_out/TAG into profiles/ as PREFIX_*, and record the bench
# step's DRAM traffic in profiles/roofline_traffic.json (keyed to the
# current kernel sources).
#   scripts/collect_final.sh r2d_final r2d
set -eu
TAG=$1; P=$2
O=gpurun_out/$TAG
D=profiles
cp $O/bench.json $D/${P}_bench_n1.json
cp $O/bench_ref.json $D/${P}_bench_reference.json
cp $O/bench_f32.json $D/${P}_bench_n1_f32.json
cp $O/bench_fma.json $D/${P}_bench_n1_fma.json
cp $O/smoke.txt $D/${P}_smoke.txt
tail -15 $O/pytest_gpu.txt > $D/${P}_pytest_gpu_summary.txt
cp $O/property_2000.txt $D/${P}_property_2000.txt
[ -f $O/memcheck.txt ] && cp $O/memcheck.txt $D/${P}_memcheck.txt
[ -f $O/racecheck.txt ] && cp $O/racecheck.txt $D/${P}_racecheck.txt
cp $O/launches.csv $D/${P}_launches_channel256_f64.csv
cat $O/ladder_*.jsonl 2>/dev/null | grep '^{' > $D/${P}_ladder.jsonl || true
for pr in f64 f32; do
  python scripts/ncu_summary.py $O/prof_step_${pr}_raw.csv 16777216 > $D/${P}_ncu_step_channel256_${pr}.json
  cp $O/prof_step_${pr}_details.txt $D/${P}_ncu_step_channel256_${pr}_details.txt
  python scripts/ncu_summary.py $O/prof_nodes_${pr}_p02_raw.csv 3429472 > $D/${P}_ncu_nodes_p02_${pr}.json
  cp $O/prof_nodes_${pr}_p02_details.txt $D/${P}_ncu_nodes_p02_${pr}_details.txt
  python scripts/ncu_stalls.py $O/prof_nodes_${pr}_p02_source.csv 12 > $D/${P}_ncu_nodes_p02_${pr}_stalls.txt
  python scripts/ncu_opmix.py $O/prof_nodes_${pr}_p02_source.csv 3429472 20 > $D/${P}_ncu_nodes_p02_${pr}_opmix.txt
done
python scripts/ncu_summary.py $O/prof_mrt_f32_raw.csv 16777216 > $D/${P}_ncu_step_channel256_mrt_f32.json
cp $O/prof_mrt_f32_details.txt $D/${P}_ncu_step_channel256_mrt_f32_details.txt
cat $O/c512_f32_tile.jsonl $O/c512_f32_auto.jsonl | grep '^{' > $D/${P}_channel512_f32_traversal.jsonl
cat $O/ncu_c512_f32_tile.csv $O/ncu_c512_f32_auto.csv > $D/${P}_ncu_channel512_f32_traversal.csv
python scripts/update_traffic.py channel256_periodic_f64_b200 $O/prof_step_f64_raw.csv $D/${P}_ncu_step_channel256_f64.json
python scripts/update_traffic.py channel256_periodic_f32_b200 $O/prof_step_f32_raw.csv $D/${P}_ncu_step_channel256_f32.json
ls $D | grep "^${P}_" | wc -l
