#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for np in 0 1; do echo "NO_PRUNE=$np"; WDD_NO_PRUNE=$np timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"colfft" -c 1 python tools/bench_live.py --config live --reps 1 2>&1 | grep -E "^  [a-z]|duration|bytes|inst|warps" | sed -E 's/\(const.*//'; done
