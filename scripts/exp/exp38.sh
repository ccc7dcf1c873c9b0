# Grouped MRT product in two row passes (10 live sums) and a shared-memory stash of the populations: occupancy A/B, parity
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_compact.py -q -x -k "mrt" 2>&1 | tail -1
for r in 1 2; do
for lib in nosplit main sp20 sp24 sp20st sp24st; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f64 --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel f64', d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel f32', d['ms'], d['frac'])"
done; done
