timeout 900 python -m pytest tests/test_gpu_slabs.py -q 2>&1 | tail -2
timeout 900 python scripts/halo_overhead.py --ranks 2,4,8 | tee gpurun_out/halo_overhead.jsonl
