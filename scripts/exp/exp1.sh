mkdir -p gpurun_out/exp1
for v in base pm2 minb12 pm2minb12 minb16; do
  if [ $v = base ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  for p in f32 f64; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision $p --variants full --steps 200 | sed "s/^/$v /" >> gpurun_out/exp1/sweep.txt 2>&1
  done
done
cat gpurun_out/exp1/sweep.txt
