# blocked traversal order on 2 M-tile domains (tuning; stdout only)
timeout 900 python -m pytest tests/test_gpu_step.py -q -k "traversal or cavity64 or random" -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_compact.py -q -x 2>&1 | tail -1
for g in "channel --n 512" "duct_z --n 1024 --length 128" "channel --n 256"; do
  for p in f32 f64; do
    timeout 300 python scripts/step_sweep.py --geometry $g --precision $p --variants full --steps 20 | cut -c1-30,225-330
  done
done
timeout 900 python scripts/step_sweep.py --geometry vessel --dims 1024,1024,2048 --variants full --steps 10 --storage compact | cut -c1-60,240-360
