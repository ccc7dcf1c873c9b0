#!/bin/bash
# fp32 MRT with packed FMUL2 products (main) vs scalar FMUL (nopack):
# parity (MRT tests, both storages) and channel 256^3 / pack p0.2 timing.
set -u
O=gpurun_out/exp53
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_compact.py tests/test_gpu_numerics.py -m gpu -q -x -k "mrt or MRT" > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
for lib in main nopack; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants mrt --steps 50 > $O/chan_${lib}_$r.jsonl 2>&1
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --precision f32 --variants mrt --steps 50 --storage compact --traversal nodes > $O/pack_${lib}_$r.jsonl 2>&1
done; done
for f in $O/*.jsonl; do echo "$f: $(tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms"], d["frac"])')"; done
ncu --set full --clock-control none -k regex:step_kernel -s 6 -c 1 -o $O/prof_mrt_f32 python scripts/step_sweep.py --variants mrt --steps 2 --precision f32 > /dev/null 2>&1
ncu -i $O/prof_mrt_f32.ncu-rep --page details > $O/prof_mrt_f32_details.txt 2>&1
ncu -i $O/prof_mrt_f32.ncu-rep --page raw --csv > $O/prof_mrt_f32_raw.csv 2>&1
rm -f $O/prof_mrt_f32.ncu-rep
