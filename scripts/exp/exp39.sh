# MRT: L2 prefetch of the tile N tiles ahead (about one wave of resident CTAs) vs none; fp64 reference and FMA arithmetic, fp32
for r in 1 2; do
for lib in main pf300 pf600 pf1200 pf2400; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  for ar in reference fma; do
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f64 --arith $ar --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'f64 $ar', d['ms'], d['frac'])"
  done
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants mrt --steps 50 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', 'f32 reference', d['ms'], d['frac'])"
done; done
