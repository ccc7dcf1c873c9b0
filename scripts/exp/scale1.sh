# large single-GPU domains (tuning/evidence; -> gpurun_out/scale1)
mkdir -p gpurun_out/scale1
O=gpurun_out/scale1/sweep.jsonl
timeout 600 python -m pytest tests/test_gpu_graph.py -q > gpurun_out/scale1/pytest_graph.txt 2>&1; tail -2 gpurun_out/scale1/pytest_graph.txt
for p in f64 f32; do
  timeout 300 python scripts/step_sweep.py --geometry cavity --n 64 --variants full --steps 1280 --precision $p >> $O 2>&1
  timeout 300 python scripts/step_sweep.py --geometry cavity --n 64 --variants full --steps 1280 --precision $p --graph >> $O 2>&1
done
timeout 600 python scripts/step_sweep.py --geometry channel --n 512 --variants full,mrt --steps 50 >> $O 2>&1
timeout 600 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --variants full --steps 50 >> $O 2>&1
timeout 600 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --variants full --steps 50 --precision f32 >> $O 2>&1
timeout 900 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 384 --variants full --steps 20 --no-perturb >> $O 2>&1
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> $O
cat $O
