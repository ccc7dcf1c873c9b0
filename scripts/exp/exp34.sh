# Grouped MRT product (distinct column products once) vs the dense product: parity, then same-box A/B over MRT occupancy
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_numerics.py tests/test_gpu_compact.py -q -x -k "mrt or MRT" 2>&1 | tail -2
for r in 1 2; do
for lib in dense main g16 g12 g24; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for prec in f64 f32; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $prec --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', '$prec', d['ms'], d['frac'])"
  done
done; done
