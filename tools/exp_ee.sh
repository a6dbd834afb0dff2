#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
WDD_FLUSH=gemm timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for f in gemm fft; do for c in live; do WDD_FLUSH=$f python tools/bench_live.py --config $c --reps 2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], '$f', round(d['frames_per_s']/1e6,2), 'frac', round(d['frac'],3), 'readout', round(d['readout_latency_us']['p50'],1))"; done; done
WDD_FLUSH=gemm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"colgemm" -c 1 python tools/bench_live.py --config live --reps 1 2>&1 | grep -E "^  [a-z]|duration|bytes|inst|tensor" | sed -E 's/\(const.*//'
