#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_simulator.py -q -x 2>&1 | tail -15
for c in medium live box; do timeout 300 python tools/bench_sim.py $c 4096; done
