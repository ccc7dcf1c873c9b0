#!/bin/bash
# Node-parallel step, nodes per thread: fp32 2 (main, 32 warps) vs 3 (npt3,
# 24 warps); fp64 1 (main, 32 warps) vs 2 (f64npt2, 16 warps).
set -u
O=gpurun_out/exp51
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_compact.py -m gpu -q -x > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
for lib in main npt3 f64npt2; do
  if [ $lib = main ]; then L=""; P=f64,f32; elif [ $lib = npt3 ]; then L=build/variants/$lib/libtlbm.so; P=f32; else L=build/variants/$lib/libtlbm.so; P=f64; fi
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.7,1.0 --precisions $P --storages nodes --steps 30 > $O/sweep_${lib}_$r.jsonl 2>$O/sweep_${lib}_$r.err
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp51/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
