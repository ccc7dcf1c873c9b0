timeout 900 python -m pytest tests/test_gpu_run.py -q -s 2>&1 | grep -E "poiseuille|passed|failed|Error|assert" | head -20
