#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for n in 1 2 4; do for acc in G spectrum; do WDD_RG_NKC=$n timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nkc=$n $acc', round(d['frames_per_s']/1e6,2), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -2 /tmp/o.txt; done; done
