# meta load before the staging barrier (tuning; stdout only)
for r in 1 2; do
for v in base late; do
  if [ $v = base ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  for p in f64 f32; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $p --variants full --steps 300 | sed "s/^/$v /" | cut -c1-40,235-320
  done
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry pack --porosity 0.5 --variants full --steps 100 | sed "s/^/$v pack /" | cut -c1-45,235-320
done; done
