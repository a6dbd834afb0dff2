#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"fft|img" -c 4 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E "^  [a-z]|duration|inst_exec" | sed -E 's/\(const.*//'
for cfg in live box; do echo "cfg=$cfg"; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fft|img" -c 4 python tools/profile_ingest.py --config $cfg --batches 2 --batch 8192 --reps 1 --synthetic-counts 2>&1 | grep -E "^  [a-z]|duration" | sed -E 's/\(const.*//' ; done
