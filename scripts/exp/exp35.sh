# Grouped MRT: parity (new grouped/dense test, MRT tests), fp32 MRT occupancy, compact MRT, same-box vs the dense product
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "mrt" 2>&1 | tail -2
for r in 1 2; do
for lib in dense main f24 f40 f48 g20; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for prec in f64 f32; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $prec --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel', '$prec', d['ms'], d['frac'])"
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --storage compact --precision $prec --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'pack0.2-compact', '$prec', d['ms'], d['frac'])"
  done
done; done
