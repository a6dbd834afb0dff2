#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for f in default fft; do for acc in G spectrum; do WDD_FLUSH=$f timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator $acc 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('live flush=$f $acc', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1), 'ingest p50', round(d['ingest_latency_us']['p50'],1))"; done; done
timeout 300 python tools/prof_cfg.py --config live --rows 64 --reps 1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"rgemm|rowfft" -c 2 -f -o gpurun_out/live_rgemm python tools/prof_cfg.py --config live --rows 64 --reps 1 > gpurun_out/ncu_rg.log 2>&1
python tools/ncu_summary.py gpurun_out/live_rgemm.ncu-rep > gpurun_out/live_rgemm.sum.txt 2>&1
python tools/ncu_hot.py gpurun_out/live_rgemm.ncu-rep 25 > gpurun_out/live_rgemm.hot.txt 2>&1
rm -f gpurun_out/live_rgemm.ncu-rep
