#!/bin/bash
# fp32 LBGK with the products paired into packed FMUL2 (lbgkpk) vs scalar
# (main): parity (fp32 step tests) and the channel / pack timings.
set -u
O=gpurun_out/exp66
mkdir -p $O
TLBM_LIB=build/variants/lbgkpk/libtlbm.so timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_compact.py tests/test_gpu_numerics.py -m gpu -q -x -k "f32 or F32 or float32 or random or cavity" > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
for lib in main lbgkpk; do
  if [ $lib = main ]; then L=""; else L=build/variants/$lib/libtlbm.so; fi
  TLBM_LIB=$L python bench.py --precision f32 --no-cpu --no-sweep --no-e2e --steps 50 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$lib', 'channel_z f32', d['ms_per_step'], d['roofline']['frac'])"
  TLBM_LIB=$L timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.6 --precisions f32 --storages nodes,blocks --steps 30 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$lib', d['case'], d['storage'], d['ms_per_step'], round(d['bu'],4))"
done; done
