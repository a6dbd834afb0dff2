#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --steps 200 > gpurun_out/r01f_bench.json 2> gpurun_out/r01f_bench.err; tail -c 3000 gpurun_out/r01f_bench.json; tail -3 gpurun_out/r01f_bench.err
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | tail -8
