mkdir -p gpurun_out/exp8
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/exp8/pytest_gpu.txt 2>&1; tail -3 gpurun_out/exp8/pytest_gpu.txt
timeout 300 python scripts/step_sweep.py --precision f32 --variants rw,prop,full --steps 200
timeout 300 python scripts/step_sweep.py --precision f32 --variants full --steps 100 --index64
for g in "channel_z --n 1024 --length 128" "channel_z --n 256 --length 256" "channel_z --n 512 --length 512"; do
  timeout 300 python scripts/step_sweep.py --geometry $g --precision f32 --variants full --steps 20
done
ncu --set full --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/exp8/f32_1024 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --precision f32 --variants full --steps 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/exp8/f32_256_idx python scripts/step_sweep.py --precision f32 --variants full --steps 2 --index64 > /dev/null 2>&1
ls gpurun_out/exp8
