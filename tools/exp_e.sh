#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu && /tmp/bw_probe
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rowfft|colfft" -c 2 -o gpurun_out/r01g_fft -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel" -s 40 -c 1 -o gpurun_out/r01g_proj -f python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
