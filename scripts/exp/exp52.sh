#!/bin/bash
# (1) fp32 large domain: channel 512^3, tile order vs y-blocked order, with
#     ncu DRAM bytes; (2) MRT on sphere packs: blocks / compact tile /
#     compact nodes, fp64 + fp32.
set -u
O=gpurun_out/exp52
mkdir -p $O
for tr in tile auto; do
  timeout 600 python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 30 --traversal $tr --no-perturb > $O/c512_f32_$tr.jsonl 2>&1
done
timeout 600 python scripts/step_sweep.py --geometry channel --n 512 --precision f64 --variants full --steps 30 --no-perturb > $O/c512_f64.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:step_kernel -s 3 -c 1 --csv --log-file $O/ncu_c512_f32_tile.csv \
   python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 2 --traversal tile --no-perturb > /dev/null 2>&1
for p in 0.2 0.5; do
for pr in f64 f32; do
  for st in "blocks tile" "compact tile" "compact nodes"; do
    set -- $st
    timeout 600 python scripts/step_sweep.py --geometry pack --porosity $p --precision $pr --variants mrt --steps 30 --storage $1 --traversal $2 > $O/mrt_p${p}_${pr}_$1_$2.jsonl 2>&1
  done
done; done
for f in $O/*.jsonl; do echo "$f: $(tail -1 $f)"; done
cat $O/ncu_c512_f32_tile.csv | tail -4
