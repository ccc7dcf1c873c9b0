# same-box A/B of the blocked traversal (stdout only)
for r in 1 2; do
for p in f64 f32; do for t in tile 16; do
  timeout 300 python scripts/step_sweep.py --geometry channel --n 512 --precision $p --variants full --steps 30 --traversal $t | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$p', 'trav=$t', d['ordered'], d['ms'], d['frac'])"
done; done; done
