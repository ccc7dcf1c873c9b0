timeout 600 python -m pytest tests/test_gpu_fma.py -q 2>&1 | tail -2
for v in mf32 mf24 mf20; do
  TLBM_LIB=build/variants/$v/libtlbm.so timeout 300 python scripts/step_sweep.py --variants mrt --arith fma --steps 100 | sed "s/^/$v /"
done
