#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in large live box; do timeout 300 python tools/bench_live.py --config $c --reps 2 > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'ingest p50', round(d['ingest_latency_us']['p50'],1), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -3 /tmp/o.txt; done
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | cut -c1-300
WDD_NVCC_EXTRA=-DWDD_TRACE python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1
python tools/trace_ctas.py large 16384 2>&1 | tail -5
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
