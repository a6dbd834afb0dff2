#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --steps 200 > gpurun_out/r01k_bench.json 2> gpurun_out/r01k_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r01k_bench.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['ms_per_step'], d['roofline']['achieved'], d['roofline']['ms_per_launch']*32, d['step_roofline']['frac'], d['e2e']['value'], d['vs_baseline'])"
