# fp32 CTA shape at 64 warps/SM, and MRT occupancy (tuning; results -> gpurun_out/exp2)
mkdir -p gpurun_out/exp2
O=gpurun_out/exp2/sweep.txt
for v in base tpc1 tpc4 minb12; do
  if [ $v = base ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants full --steps 200 | sed "s/^/$v /" >> $O 2>&1
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f32 --variants full --steps 100 --geometry pack --porosity 0.5 | sed "s/^/$v /" >> $O 2>&1
done
for v in base mrt8 mrt6; do
  if [ $v = base ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  for p in f32 f64; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $p --variants mrt --steps 100 | sed "s/^/$v /" >> $O 2>&1
  done
done
cat $O
