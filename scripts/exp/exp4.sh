mkdir -p gpurun_out/exp4
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/exp4/pytest_gpu.txt 2>&1; tail -5 gpurun_out/exp4/pytest_gpu.txt
timeout 600 python -m pytest tests/test_gpu_fma.py -q -s 2>&1 | grep "rel f" > gpurun_out/exp4/fma_rel.txt
python bench.py > gpurun_out/exp4/bench.json 2> gpurun_out/exp4/bench.err; cat gpurun_out/exp4/bench.json
python bench.py --precision f32 --no-cpu > gpurun_out/exp4/bench_f32.json 2>> gpurun_out/exp4/bench.err; cat gpurun_out/exp4/bench_f32.json
cat gpurun_out/exp4/fma_rel.txt
