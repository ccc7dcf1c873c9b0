mkdir -p gpurun_out/exp5
timeout 120 compute-sanitizer --tool memcheck python scripts/exp/idx64.py f32 lbgk 2>&1 | tail -3
TLBM_LIB=build/variants/idx40/libtlbm.so timeout 120 compute-sanitizer --tool memcheck python scripts/exp/idx64.py f32 lbgk 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/exp5/pytest_gpu.txt 2>&1; tail -3 gpurun_out/exp5/pytest_gpu.txt
