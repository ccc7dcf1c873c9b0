#!/bin/bash
# e2e setup phases; bench e2e with pinned tags and a single initial
# equilibrium; GPU tests touching the tiler / solver init / slabs.
set -u
O=gpurun_out/exp58
mkdir -p $O
python scripts/e2e_phases.py --reps 3 > $O/phases.jsonl 2>&1
cat $O/phases.jsonl
timeout 1500 python -m pytest tests/test_gpu_tiler.py tests/test_gpu_step.py tests/test_gpu_slabs.py tests/test_gpu_run.py -m gpu -q -x > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
python bench.py --no-sweep --no-cpu > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e'])"
