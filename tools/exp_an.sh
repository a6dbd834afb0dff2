#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -s 2>&1 | grep -E "passed|failed|^large|^live|^box"
for c in large; do timeout 300 python tools/bench_live.py --config $c --reps 3 > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'ingest p50', round(d['ingest_latency_us']['p50'],1), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -3 /tmp/o.txt; done
