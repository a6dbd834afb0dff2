#!/bin/bash
WDD_NVCC_EXTRA=-DWDD_TRACE python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1
python tools/trace_proj.py large 8192 600 > gpurun_out/trace_large.txt 2>&1
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
