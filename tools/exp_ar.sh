#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -1
python bench.py --steps 300 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('medium', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"
for c in large live box; do timeout 300 python tools/bench_live.py --config $c --reps 2 > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -3 /tmp/o.txt; done
ncu --metrics gpu__time_duration.sum -k regex:rowfft -c 3 python tools/prof_cfg.py --config live --rows 64 --reps 1 2>/dev/null | grep -E "rowfft|duration" | head -4
ncu --metrics gpu__time_duration.sum -k regex:rowfft -c 1 python tools/prof_cfg.py --config large --rows 256 --reps 1 2>/dev/null | grep -E "duration" | head -2
