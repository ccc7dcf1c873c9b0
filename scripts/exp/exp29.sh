# traversal auto: fp32 blocks ordered, fp64 / compact tile order (stdout only)
for g in "channel --n 512" "duct_z --n 1024 --length 128"; do
  for p in f32 f64; do
    timeout 300 python scripts/step_sweep.py --geometry $g --precision $p --variants full --steps 20 | cut -c1-30,225-330
  done
done
