# Moment-space FMA MRT (final form: no dense FMA fallback in the kernel, 24 warps/SM): parity + timing
timeout 900 python -m pytest tests/test_gpu_fma.py tests/test_gpu_step.py tests/test_gpu_compact.py -q -x -k "fma or mrt" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_property.py -q -x 2>&1 | tail -1
for r in 1 2; do
  for ar in fma reference; do
  timeout 300 python scripts/step_sweep.py --precision f64 --arith $ar --variants full,mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('channel', '$ar', d['variant'], d['ms'], d['frac'])"
  timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --storage compact --arith $ar --variants full,mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('pack0.2-compact', '$ar', d['variant'], d['ms'], d['frac'])"
done; done
