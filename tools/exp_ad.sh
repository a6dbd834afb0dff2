#!/bin/bash
WDD_NVCC_EXTRA=-DWDD_TRACE python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1
python tools/trace_ctas.py large 16384 2>&1 | tail -8
python tools/trace_ctas.py medium 512 2>&1 | tail -8
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
