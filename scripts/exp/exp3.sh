# arithmetic modes x collision x dtype, MRT occupancy (tuning; -> gpurun_out/exp3)
mkdir -p gpurun_out/exp3
O=gpurun_out/exp3/sweep.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp3/pytest_gpu.txt 2>&1; tail -3 gpurun_out/exp3/pytest_gpu.txt
timeout 600 python -m pytest tests/test_gpu_fma.py -q -s 2>&1 | grep "rel f" > gpurun_out/exp3/fma_rel.txt
for ar in reference fma; do for p in f64 f32; do
  timeout 300 python scripts/step_sweep.py --precision $p --variants full,mrt --steps 200 --arith $ar >> $O 2>&1
done; done
for v in mrtw16 mrtw24 mrtw32; do for ar in reference fma; do for p in f64 f32; do
  TLBM_LIB=build/variants/$v/libtlbm.so timeout 300 python scripts/step_sweep.py --precision $p --variants mrt --steps 100 --arith $ar | sed "s/^/$v /" >> $O 2>&1
done; done; done
cat $O gpurun_out/exp3/fma_rel.txt
