#!/bin/bash
# fp64 MRT (reference arithmetic) on the node-parallel step with two nodes per
# thread (mrtnpt2, 12 warps/SM, 166 registers) vs one (main, 16 warps; and
# mrtnpt1w12 at 12 warps), channel 256^3 and packs p0.2 / p0.5, against the
# block-store MRT kernel.
set -u
O=gpurun_out/exp56
mkdir -p $O
TLBM_LIB=build/variants/mrtnpt2/libtlbm.so timeout 900 python -m pytest tests/test_gpu_compact.py -m gpu -q -x -k "mrt or equals" > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
for lib in main mrtnpt2 mrtnpt1w12; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  echo "== $lib" >> $O/runs_$r.txt
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry channel --n 256 --variants mrt --steps 30 --storage compact --traversal nodes >> $O/runs_$r.txt 2>&1
  for p in 0.2 0.5; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity $p --variants mrt --steps 30 --storage compact --traversal nodes >> $O/runs_$r.txt 2>&1
  done
  if [ $lib = main ]; then
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry channel --n 256 --variants mrt --steps 30 >> $O/runs_$r.txt 2>&1
  fi
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp56/runs_*.txt')):
    for l in open(f):
        if l.startswith('=='): print(l.strip()); continue
        try: d=json.loads(l)
        except Exception: continue
        print(' ', d['geometry'], d.get('storage'), d['ms'], d['frac'])
PY
