#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for tpc in 0 1 2; do WDD_COLFFT_TPC=$tpc python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('medium tpc=$tpc', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"; done
for tpc in 0 1 4 16; do WDD_COLFFT_TPC=$tpc python tools/bench_live.py --config live --reps 2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('live tpc=$tpc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))"; done
