#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('default', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"
for mf in 4 8 12 24; do WDD_PROJ_MIN_FRAMES=$mf python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mf=$mf(no wide)', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"; done
