#!/bin/bash
# Slab-decomposition overhead on one GPU for the porosity-0.2 pack with the
# node-parallel step (storage auto) and with blocks, fp64 and fp32.
set -u
O=gpurun_out/exp67
mkdir -p $O
for st in auto blocks; do
for pr in f64 f32; do
  timeout 900 python scripts/halo_overhead.py --geometry pack --porosity 0.2 --storage $st --precision $pr --ranks 2,4,8 --steps 30 >> $O/halo_pack.jsonl 2>> $O/err.txt
done; done
timeout 900 python scripts/halo_overhead.py --ranks 2,4,8 --steps 30 >> $O/halo_channel.jsonl 2>> $O/err.txt
cat $O/*.jsonl
tail -5 $O/err.txt
