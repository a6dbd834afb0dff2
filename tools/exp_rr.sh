#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for acc in G spectrum; do timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('live $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1), 'ingest p50', round(d['ingest_latency_us']['p50'],1))"; done
ncu --set full --clock-control none --import-source on -k regex:"rgemm" -s 1 -c 1 -f -o gpurun_out/live_rgemm3 python tools/prof_cfg.py --config live --rows 128 --readout-rows 64 --reps 1 > gpurun_out/ncu_rg3.log 2>&1
python tools/ncu_summary.py gpurun_out/live_rgemm3.ncu-rep > gpurun_out/live_rgemm3.sum.txt 2>&1
python tools/ncu_hot.py gpurun_out/live_rgemm3.ncu-rep 25 > gpurun_out/live_rgemm3.hot.txt 2>&1
