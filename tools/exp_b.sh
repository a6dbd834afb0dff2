#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_ingest.py --config medium --batches 32 --batch 512 --reps 3 --synthetic-counts 2>&1 | tail -2
for mf in 8 16 32; do echo "MIN_FRAMES=$mf"; WDD_PROJ_MIN_FRAMES=$mf python bench.py --steps 100 --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']/1e6, d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,2) for k,v in d['kernels'].items()})"; done
python bench.py --steps 200 --no-cpu-baseline > gpurun_out/r01d_bench.json 2>&1; tail -c 2500 gpurun_out/r01d_bench.json
