#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for acc in G spectrum; do timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('live $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1), 'ingest p50', round(d['ingest_latency_us']['p50'],1))"; done
WDD_NVCC_EXTRA=-DWDD_TRACE python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1
python tools/trace_rgemm.py G | tail -20
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
