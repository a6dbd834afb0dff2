#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { for c in large box; do timeout 300 python tools/bench_live.py --config $c --reps 2 > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 $c', round(d['frames_per_s']/1e6,2), 'readout', round(d['readout_latency_us']['p50'],1))" || tail -2 /tmp/o.txt; done; }
run base
for rf in 2,256 3,256 3,128 4,128; do WDD_ROWFFT=$rf run rowfft=$rf; done
for cf in 3,256 4,128 4,256 5,512; do WDD_COLFFT=$cf run colfft=$cf; done
