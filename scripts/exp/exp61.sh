#!/bin/bash
# fp64 MRT at one tile per CTA (main now): MRT parity tests and timing.
set -u
O=gpurun_out/exp61
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_fma.py tests/test_gpu_slabs.py tests/test_gpu_graph.py tests/test_gpu_ladder.py -m gpu -q -x > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
  for ar in reference fma; do
  timeout 300 python scripts/step_sweep.py --precision f64 --arith $ar --variants full,mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$ar', d['variant'], d['ms'], d['frac'])"
  done
done
