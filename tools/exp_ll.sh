#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_spectrum_mode.py -x -q 2>&1 | tail -15
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for acc in G spectrum; do for cfg in live large box; do python tools/bench_live.py --config $cfg --reps 2 --accumulator $acc 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1), 'ingest p50', round(d['ingest_latency_us']['p50'],1))"; done; done
