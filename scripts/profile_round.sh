#!/bin/bash
# Full evidence pass on the GPU box (via gpurun): bench lines (fp64, fp32),
# step ladders, ncu launch list, ncu --set full of the step kernel (fp64,
# fp32, MRT reference and FMA arithmetic), sparse DRAM bytes, porosity sweep,
# sanitizers.  Outputs under gpurun_out/$TAG/.
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --precision f32 --no-cpu --no-sweep > $O/bench_f32.json 2>> $O/bench.err
python bench.py --arith fma --no-cpu --no-sweep > $O/bench_fma.json 2>> $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench.err
python scripts/step_sweep.py --variants rw,prop,full,mrt > $O/ladder_f64.jsonl 2>/dev/null
python scripts/step_sweep.py --variants full,mrt --arith fma > $O/ladder_f64_fma.jsonl 2>/dev/null
python scripts/step_sweep.py --variants rw,prop,full,mrt --precision f32 > $O/ladder_f32.jsonl 2>/dev/null
python scripts/step_sweep.py --geometry cavity --n 64 --variants full --steps 1000 > $O/cavity64.jsonl 2>/dev/null
python scripts/step_sweep.py --geometry cavity --n 64 --variants full --steps 1000 --precision f32 >> $O/cavity64.jsonl 2>/dev/null
python scripts/porosity_sweep.py --vessel --cavity --storages blocks,compact > $O/sweep.jsonl 2> $O/sweep.err
python scripts/halo_overhead.py --ranks 2,4,8 --steps 60 > $O/halo_overhead.jsonl 2>/dev/null
python scripts/step_sweep.py --geometry cavity --n 64 --variants full --steps 1280 --graph >> $O/cavity64.jsonl 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
for p in f64 f32; do
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
      -o $O/prof_step_$p python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-sweep --precision $p > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
    -o $O/prof_step_mrt python scripts/step_sweep.py --variants mrt --steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
    -o $O/prof_step_mrt_fma python scripts/step_sweep.py --variants mrt --steps 2 --arith fma > /dev/null 2>&1
for p in 0.2 0.5 0.9; do
  for st in blocks compact; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:step_kernel -s 5 -c 1 --csv --log-file $O/ncu_sparse_${st}_p$p.csv \
      python scripts/porosity_sweep.py --porosities $p --precisions f64 --storages $st --steps 3 --warmup 5 > /dev/null 2>&1
  done
done
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_step_compact_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions f64 --storages compact --steps 3 --warmup 5 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:step_kernel -s 5 -c 1 --csv --log-file $O/ncu_sparse_vessel.csv \
    python scripts/porosity_sweep.py --porosities "" --vessel --precisions f64 --steps 3 --warmup 5 > /dev/null 2>&1
# gpurun copies back at most 64 MiB: keep text/CSV exports of every full
# capture and only the fp64 step report itself
for r in $O/prof_step_*.ncu-rep; do
  ncu -i $r --page details > ${r%.ncu-rep}_details.txt 2>&1
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>&1
  [ "$r" = "$O/prof_step_f64.ncu-rep" ] || rm -f $r
done
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_small.py > $O/memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python scripts/sanitize_small.py > $O/racecheck.txt 2>&1
tail -2 $O/memcheck.txt $O/racecheck.txt
cat $O/bench.json $O/bench_f32.json $O/bench_fma.json
ls $O
