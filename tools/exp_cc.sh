#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for f in gemm fft; do
WDD_FLUSH=$f python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('medium $f', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"
for c in live box; do WDD_FLUSH=$f python tools/bench_live.py --config $c --reps 2 $( [ $c = box ] && echo --batch 16384 ) 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], '$f', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))"; done; done
