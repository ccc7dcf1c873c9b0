set -u
python bench.py --steps 100 2>&1 | tail -1 | cut -c1-200
python bench.py --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --n 64 --transport gloo 2>&1 | grep -E '^\{|Error|error' | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --impl reference 2>&1 | grep -E '^\{|Error|error' | cut -c1-400
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_small.py 2>&1 | tail -5
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_small.py 2>&1 | tail -5
