timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed|FAILED|Error" | head -20
python scripts/step_sweep.py --variants rw,prop,full,mrt 2>&1 | grep '{'
python scripts/step_sweep.py --variants rw,prop,full,mrt --precision f32 2>&1 | grep '{'
