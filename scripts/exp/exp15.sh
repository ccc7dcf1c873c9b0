timeout 900 python -m pytest tests/test_gpu_slabs.py -q 2>&1 | tail -2
python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29615 bench.py --gpus 3 --steps 10 --warmup 3 --edge 64 2>&1 | grep -E '^\{|Error|error' | cut -c1-200
