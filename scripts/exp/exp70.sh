#!/bin/bash
# 12-byte node records (source ranks only for tile-crossing pulls; rank bytes
# of the tile for the rest; own rank from the index) vs the 20-byte records
# (build/old_tree: the previous commit's package and library).
set -u
O=gpurun_out/exp70
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_compact.py tests/test_gpu_slabs.py tests/test_gpu_parity_full.py -m gpu -q -x -k "nodes or compact or records or equals or p02 or auto" > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
for r in 1 2; do
  timeout 600 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.8 --vessel --precisions f64,f32 --storages nodes --steps 30 > $O/sweep_new_$r.jsonl 2>$O/err_new_$r.txt
  timeout 600 python build/old_tree/scripts/porosity_sweep.py --porosities 0.2,0.5,0.8 --vessel --precisions f64,f32 --storages nodes --steps 30 > $O/sweep_old_$r.jsonl 2>$O/err_old_$r.txt
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/exp70/sweep_*.jsonl')):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d['case'], d['precision'], d['storage'], round(d['ms_per_step'],4), round(d['bu'],4))
PY
for pr in f64 f32; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:step_kernel -s 5 -c 1 --csv --log-file $O/ncu_new_$pr.csv \
  python scripts/porosity_sweep.py --porosities 0.2 --precisions $pr --storages nodes --steps 3 --warmup 5 > /dev/null 2>&1
grep dram__ $O/ncu_new_$pr.csv | awk -F'","' '{print "'$pr'", $13, $15}'
done
