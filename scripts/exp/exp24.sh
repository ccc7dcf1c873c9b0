for v in base c48 c64; do
  if [ $v = base ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  TLBM_LIB=$L timeout 900 python scripts/porosity_sweep.py --porosities 0.2,0.5 --storages compact --precisions f32 --steps 30 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('$v', d['case'], d['precision'], d['storage'], round(d['mlups']), round(d['bu'],3))
    else: print(l.strip())"
done
