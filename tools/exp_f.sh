#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu && /tmp/bw_probe
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 200 > gpurun_out/r01h_bench.json 2> gpurun_out/r01h_bench.err; tail -c 3000 gpurun_out/r01h_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fft|readout|img_|flush|rowdft" -c 8 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E "  [a-z].*kernel|duration|bytes" | head -40
