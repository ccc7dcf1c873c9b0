mkdir -p gpurun_out/exp16
timeout 900 python -m pytest tests/test_gpu_compact.py -q -x > gpurun_out/exp16/pytest.txt 2>&1; tail -5 gpurun_out/exp16/pytest.txt
timeout 900 python scripts/porosity_sweep.py --porosities 0.2,0.5,0.9,1.0 --storages blocks,compact --steps 30 > gpurun_out/exp16/sweep.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/exp16/sweep.jsonl"):
    if not l.startswith("{"): print(l.strip()); continue
    d = json.loads(l); print(d["case"], d["precision"], d["storage"], round(d["mlups"]), round(d["bu"], 3))
PY
for p in 0.2 0.5; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:step_kernel -s 5 -c 1 --csv python scripts/porosity_sweep.py --porosities $p --precisions f64 --storages compact --steps 3 --warmup 5 2>&1 | grep -E '"dram|"gpu__' | sed -E 's/.*"(dram__bytes_[a-z]+.sum|gpu__time_duration.sum)","[a-z]+","([0-9.]+)"/\1 \2/' | sed "s/^/compact p$p: /"
done
