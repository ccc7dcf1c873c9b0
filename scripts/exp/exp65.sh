#!/bin/bash
# Full GPU suite + bench after the MRT occupancy / e2e changes.
set -u
O=gpurun_out/exp65
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
python bench.py --no-sweep --no-cpu > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['phases'])"
python scripts/step_sweep.py --variants rw,prop,full,mrt --steps 50 > $O/ladder_f64.jsonl 2>/dev/null
python scripts/step_sweep.py --variants full,mrt --arith fma --steps 50 > $O/ladder_f64_fma.jsonl 2>/dev/null
python scripts/step_sweep.py --variants rw,prop,full,mrt --precision f32 --steps 50 > $O/ladder_f32.jsonl 2>/dev/null
cat $O/ladder_*.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['precision'], d['arith'], d['variant'], d['ms'], d['frac'])
    except Exception: pass"
