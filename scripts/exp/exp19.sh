mkdir -p gpurun_out/exp19
for st in compact blocks; do for p in 0.2 0.9; do
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 -o gpurun_out/exp19/${st}_p$p python scripts/porosity_sweep.py --porosities $p --precisions f64 --storages $st --steps 3 --warmup 5 > /dev/null 2>&1
done; done
ls gpurun_out/exp19
