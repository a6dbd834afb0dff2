#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { echo "ROW=$1 COL=$2"; WDD_ROWFFT=$1 WDD_COLFFT=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fft" -c 2 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E "duration" ; }
run -1,0 -1,0
run 4,128 4,128
run 3,64 3,64
run 5,512 5,512
run 4,256 4,256
run 3,128 3,128
