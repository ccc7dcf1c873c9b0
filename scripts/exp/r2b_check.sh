set -u
O=gpurun_out/r2b_check
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
for p in 0.2; do for st in blocks compact; do for pr in f32 f64; do
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
    -o $O/prof_${pr}_${st}_p$p python scripts/porosity_sweep.py --porosities $p --precisions $pr --storages $st --steps 3 --warmup 5 > /dev/null 2>&1
ncu -i $O/prof_${pr}_${st}_p$p.ncu-rep --page details > $O/prof_${pr}_${st}_p${p}_details.txt 2>&1
ncu -i $O/prof_${pr}_${st}_p$p.ncu-rep --page source --csv > $O/prof_${pr}_${st}_p${p}_source.csv 2>&1
done; done; done
ls -la $O
