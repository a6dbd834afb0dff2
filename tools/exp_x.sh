#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/bench_live.py --config live > gpurun_out/r01x_live.json 2>&1; tail -1 gpurun_out/r01x_live.json
python tools/bench_live.py --config large --batch 65536 > gpurun_out/r01x_large.json 2>&1; tail -1 gpurun_out/r01x_large.json
python tools/bench_live.py --config box --batch 16384 --reps 2 > gpurun_out/r01x_box.json 2>&1; tail -1 gpurun_out/r01x_box.json
