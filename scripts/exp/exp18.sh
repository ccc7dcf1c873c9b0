mkdir -p gpurun_out/exp18
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 -o gpurun_out/exp18/compact_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions f64 --storages compact --steps 3 --warmup 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 -o gpurun_out/exp18/blocks_p02 python scripts/porosity_sweep.py --porosities 0.2 --precisions f64 --storages blocks --steps 3 --warmup 5 > /dev/null 2>&1
ls gpurun_out/exp18
