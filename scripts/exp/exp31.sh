# packed compact kernel vs slot-mapped (stdout only)
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_property.py -q -x 2>&1 | tail -1
for p in 0.2 0.5 0.9; do for prec in f64 f32; do for pk in "" "--no-pack"; do
  timeout 300 python scripts/step_sweep.py --geometry pack --porosity $p --precision $prec --storage compact --variants full --steps 50 $pk | cut -c1-10,200-420 | sed "s/^/p$p /"
done; done; done
