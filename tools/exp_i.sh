#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
j() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), 'proj_us', round(d['roofline']['ms_per_launch']*d['roofline']['launches_per_step']*1e3,1), round(d['roofline']['achieved']))"; }
for b in 256 512 1024 2048 16384; do python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 --batch $b 2>/dev/null | j "batch=$b"; done
for b in 512 2048; do WDD_PROJ_NO_PDLWAIT=1 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 --batch $b 2>/dev/null | j "nowait batch=$b"; done
WDD_PROJ_MIN_FRAMES=0 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 --batch 16384 2>/dev/null | j "allSM batch=16384"
