#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 200 > gpurun_out/r01e_bench.json 2>&1; tail -c 2800 gpurun_out/r01e_bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rowfft|colfft|img_|readout" -c 5 -o gpurun_out/r01e_acc -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/r01e_acc.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|DRAM Throughput|Memory Throughput|Compute \(SM\) Throughput|Achieved Occupancy|Registers Per Thread)"' | cut -d, -f5,15- | head -40
