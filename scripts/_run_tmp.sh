set -u
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --edge 64 --transport gloo 2>&1 | grep -E '^\{|Error|error' | cut -c1-1500
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 3 --steps 20 --warmup 3 --edge 64 --transport gloo 2>&1 | grep -E '^\{|Error|error' | cut -c1-300
python bench.py --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
