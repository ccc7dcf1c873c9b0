# Final check of the committed code: smoke, full pytest -m gpu, default bench line
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final/pytest_gpu.txt 2>&1; tail -1 gpurun_out/final/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -c 400 gpurun_out/final/bench.json
