timeout 900 python -m pytest tests/test_gpu_compact.py -q -x 2>&1 | tail -2
timeout 900 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.9 --storages compact,blocks --precisions f64 --steps 30 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['case'], d['precision'], d['storage'], round(d['mlups']), round(d['bu'],3))
    else: print(l.strip())"
