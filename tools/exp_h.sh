#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r01i_bench.json 2> gpurun_out/r01i_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r01i_bench.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['ms_per_step'], d['roofline']['achieved'], d['roofline']['ms_per_launch']*32)"
for mf in 16 64; do WDD_PROJ_MIN_FRAMES=$mf python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mf=$mf', d['value']/1e6, d['ms_per_step'], d['roofline']['achieved'], d['roofline']['ms_per_launch']*32)"; done
