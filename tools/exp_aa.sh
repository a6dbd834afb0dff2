#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"fft|img|readout" -c 5 python tools/bench_live.py --config live --reps 1 2>&1 | grep -E "^  [a-z]|duration|bytes|inst" | sed -E 's/\(const.*//'
