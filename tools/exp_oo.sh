#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in default fused cufft; do WDD_IMG=$m python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('medium img=$m', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"; done
for m in default fused cufft; do for cfg in large live; do WDD_IMG=$m python tools/bench_live.py --config $cfg --reps 2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg img=$m', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1), 'ingest p50', round(d['ingest_latency_us']['p50'],1), 'host', round(d['host_us_per_ingest_call']['p50'],1))"; done; done
python tools/bench_live.py --config box --reps 2 2>&1 | tail -1
