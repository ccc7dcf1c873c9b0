# FMA-arithmetic MRT in moment space (pair sums/differences, integer basis) vs the dense FMA product: parity, occupancy A/B
timeout 900 python -m pytest tests/test_gpu_fma.py tests/test_gpu_step.py -q -x -k "fma or mrt" 2>&1 | tail -2
for r in 1 2; do
for lib in dfma main m16 m24 nd20 nd24; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f64 --arith fma --variants mrt,full --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'channel', d['variant'], d['ms'], d['frac'])"
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.2 --storage compact --arith fma --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'pack0.2-compact', d['variant'], d['ms'], d['frac'])"
done; done
