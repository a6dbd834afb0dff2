#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rowfft|colfft|img_" -c 4 -o gpurun_out/r01j_fft -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/r01j_fft.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|DRAM Throughput|Compute \(SM\) Throughput|Achieved Occupancy|Executed Ipc Active|Issue Slots Busy)"' | cut -d, -f5,15- 
