mkdir -p gpurun_out/exp10
timeout 600 python -m pytest tests/test_gpu_checkpoint.py tests/test_gpu_slabs.py tests/test_gpu_graph.py -q > gpurun_out/exp10/pytest.txt 2>&1; tail -15 gpurun_out/exp10/pytest.txt
