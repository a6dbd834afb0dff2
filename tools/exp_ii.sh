#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for nw in 0 1; do WDD_PROJ_NO_PDLWAIT=$nw python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nowait=$nw', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), 'proj', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1))"; done
WDD_PROJ_NO_PDLWAIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
