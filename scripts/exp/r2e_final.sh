#!/bin/bash
# Round-2 final evidence pass (run on the final code): smoke, pytest -m gpu,
# bench lines (default, reference arm, fp32, fma), ncu launch list and full
# captures (bench step f64/f32 -> roofline traffic; node-parallel p0.2;
# fp32 MRT), fp32 512^3 tile vs y-blocked DRAM bytes, property test x2000
# (compute-sanitizer is closed on this pool; r2c/r2d ran it).
set -u
TAG=${1:-r2e_final}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench.err
python bench.py --precision f32 --no-cpu --no-sweep > $O/bench_f32.json 2>> $O/bench.err
python bench.py --arith fma --no-cpu --no-sweep > $O/bench_fma.json 2>> $O/bench.err
python scripts/step_sweep.py --variants rw,prop,full,mrt --steps 50 > $O/ladder_f64.jsonl 2>/dev/null
python scripts/step_sweep.py --variants full,mrt --arith fma --steps 50 > $O/ladder_f64_fma.jsonl 2>/dev/null
python scripts/step_sweep.py --variants rw,prop,full,mrt --precision f32 --steps 50 > $O/ladder_f32.jsonl 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
for pr in f64 f32; do
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
      -o $O/prof_step_$pr python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-sweep --precision $pr > /dev/null 2>&1
  ncu -i $O/prof_step_$pr.ncu-rep --page raw --csv > $O/prof_step_${pr}_raw.csv 2>&1
  ncu -i $O/prof_step_$pr.ncu-rep --page details > $O/prof_step_${pr}_details.txt 2>&1
  [ $pr = f64 ] || rm -f $O/prof_step_$pr.ncu-rep
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_nodes_${pr}_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages nodes --steps 3 --warmup 5 > /dev/null 2>&1
  ncu -i $O/prof_nodes_${pr}_p02.ncu-rep --page details > $O/prof_nodes_${pr}_p02_details.txt 2>&1
  ncu -i $O/prof_nodes_${pr}_p02.ncu-rep --page raw --csv > $O/prof_nodes_${pr}_p02_raw.csv 2>&1
  ncu -i $O/prof_nodes_${pr}_p02.ncu-rep --page source --csv > $O/prof_nodes_${pr}_p02_source.csv 2>&1
  rm -f $O/prof_nodes_${pr}_p02.ncu-rep
done
ncu --set full --clock-control none -k regex:step_kernel -s 6 -c 1 -o $O/prof_mrt_f32 python scripts/step_sweep.py --variants mrt --steps 2 --precision f32 > /dev/null 2>&1
ncu -i $O/prof_mrt_f32.ncu-rep --page details > $O/prof_mrt_f32_details.txt 2>&1
ncu -i $O/prof_mrt_f32.ncu-rep --page raw --csv > $O/prof_mrt_f32_raw.csv 2>&1
rm -f $O/prof_mrt_f32.ncu-rep
for tr in tile auto; do
  timeout 600 python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 30 --traversal $tr --no-perturb > $O/c512_f32_$tr.jsonl 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:step_kernel -s 3 -c 1 --csv --log-file $O/ncu_c512_f32_$tr.csv \
     python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 2 --traversal $tr --no-perturb > /dev/null 2>&1
done
TLBM_PROPERTY_EXAMPLES=2000 timeout 2400 python -m pytest tests/test_gpu_property.py -m gpu -q --hypothesis-show-statistics > $O/property_2000.txt 2>&1
tail -3 $O/property_2000.txt
du -sh $O
ls -la $O/*.ncu-rep
