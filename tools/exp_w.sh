#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
j() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"; }
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | j fused
WDD_IMG_UNFUSED=1 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | j unfused
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"img" -c 2 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E "img|duration" | sed -E 's/\(const.*//'
