#!/bin/bash
# Round-2 evidence pass: smoke, pytest -m gpu, bench (default + reference arm),
# nodes porosity sweep, ncu launch list + step captures.
set -u
O=gpurun_out/r2b_full
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench.err
tail -c 1500 $O/bench.json
timeout 900 python scripts/porosity_sweep.py --vessel --storages blocks,compact,nodes --steps 50 > $O/sweep.jsonl 2> $O/sweep.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
for pr in f64 f32; do
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
      -o $O/prof_step_$pr python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-sweep --precision $pr > /dev/null 2>&1
  ncu -i $O/prof_step_$pr.ncu-rep --page raw --csv > $O/prof_step_${pr}_raw.csv 2>&1
  ncu -i $O/prof_step_$pr.ncu-rep --page details > $O/prof_step_${pr}_details.txt 2>&1
  rm -f $O/prof_step_$pr.ncu-rep
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_nodes_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages nodes --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_nodes_${pr}_p02.ncu-rep --page details > $O/prof_nodes_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_nodes_${pr}_p02.ncu-rep --page raw --csv > $O/prof_nodes_${pr}_p02_raw.csv 2>&1
  ncu -i $O/prof_nodes_${pr}_p02.ncu-rep --page source --csv > $O/prof_nodes_${pr}_p02_source.csv 2>&1
  rm -f $O/prof_nodes_${pr}_p02.ncu-rep
done
du -sh $O
