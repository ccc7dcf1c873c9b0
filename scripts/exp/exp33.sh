# same-box A/B of the blocked traversal, auto band height (stdout only)
for r in 1 2; do
for g in "channel --n 512" "duct_z --n 1024 --length 128"; do for t in tile auto; do
  timeout 300 python scripts/step_sweep.py --geometry $g --precision f32 --variants full --steps 30 --traversal $t | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$g', 'trav=$t', d['ordered'], d['ms'], d['frac'])"
done; done; done
