#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spectrum_mode.py -q -x 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "live" 2>&1 | tail -1
for acc in G spectrum; do timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('live $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -2 /tmp/o.txt; done
ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum -k regex:rgemm -s 1 -c 1 python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1 2>/dev/null | grep -E "duration|conflicts"
