for v in ptr32 ptr64; do
  TLBM_LIB=build/variants/$v/libtlbm.so timeout 120 compute-sanitizer --tool memcheck python scripts/exp/idx64.py f32 lbgk 2>&1 | tail -2 | sed "s/^/$v /"
  TLBM_LIB=build/variants/$v/libtlbm.so timeout 300 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --precision f32 --variants full --steps 20 | sed "s/^/$v /"
  TLBM_LIB=build/variants/$v/libtlbm.so timeout 300 python scripts/step_sweep.py --precision f32 --variants full --steps 100 --index64 | sed "s/^/$v /"
done
TLBM_LIB=build/variants/ptr64/libtlbm.so timeout 120 compute-sanitizer --tool memcheck python scripts/exp/idx64.py f64 lbgk 2>&1 | tail -2
TLBM_LIB=build/variants/ptr64/libtlbm.so timeout 300 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --precision f64 --variants full --steps 20 | sed "s/^/ptr64 /"
TLBM_LIB=build/variants/ptr64/libtlbm.so timeout 300 python scripts/step_sweep.py --precision f64 --variants full,mrt --steps 100 --index64 | sed "s/^/ptr64 /"
