# N>1 bench code path on one GPU (ranks share cuda:0; timing meaningless)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --edge 128 2>&1 | grep -E '^\{|Error|error' | cut -c1-400
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --edge 128 --precision f32 2>&1 | grep -E '^\{|Error|error' | cut -c1-400
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 --steps 10 --warmup 3 --edge 64 --transport gloo 2>&1 | grep -E '^\{|Error|error' | cut -c1-400
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 2 --steps 10 --warmup 3 --impl reference --edge 64 2>&1 | grep -E '^\{|Error|error' | cut -c1-300
