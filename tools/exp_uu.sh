#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3 4; do timeout 300 python tools/bench_live.py --config live --reps 2 --accumulator G > /tmp/bl_$i.txt 2>&1; echo "rc=$?"; tail -c 300 /tmp/bl_$i.txt; echo; done
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spectrum_mode.py -x -q 2>&1 | tail -1; done
timeout 300 python tools/bench_live.py --config large --reps 2 2>&1 | tail -c 400
timeout 300 python tools/bench_live.py --config box --reps 1 2>&1 | tail -c 400
