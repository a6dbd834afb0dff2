#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for ab in 0 2 4 8 6 12 14; do echo "ABLATE=$ab"; WDD_COLFFT_V=1 WDD_ABLATE=$ab timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"colfft" -c 1 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E "duration|inst_exec"; done
