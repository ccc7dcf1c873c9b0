mkdir -p gpurun_out/exp22
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/exp22/pytest_gpu.txt 2>&1; tail -3 gpurun_out/exp22/pytest_gpu.txt
timeout 1500 python scripts/porosity_sweep.py --vessel --storages blocks,compact > gpurun_out/exp22/sweep.jsonl 2> gpurun_out/exp22/sweep.err
python - <<'PY'
import json
for l in open("gpurun_out/exp22/sweep.jsonl"):
    if not l.startswith("{"): continue
    d = json.loads(l); print(d["case"], d["precision"], d["storage"], round(d["mlups"]), round(d["bu"], 3))
PY
for p in 0.2 0.5 0.9; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:step_kernel -s 5 -c 1 --csv --log-file gpurun_out/exp22/ncu_compact_p$p.csv python scripts/porosity_sweep.py --porosities $p --precisions f64 --storages compact --steps 3 --warmup 5 > /dev/null 2>&1
done
ls gpurun_out/exp22
