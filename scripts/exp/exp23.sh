# BASELINE config 5's sparse 2048x1024x1024 vessel tree on ONE GPU (75 GB fp64)
mkdir -p gpurun_out/exp23
for st in blocks compact; do
  timeout 1200 python scripts/step_sweep.py --geometry vessel --dims 1024,1024,2048 --variants full --steps 10 --storage $st | tee -a gpurun_out/exp23/vessel_big.jsonl | cut -c1-330
done
nvidia-smi --query-gpu=memory.total --format=csv
