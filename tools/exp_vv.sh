#!/bin/bash
WDD_NVCC_EXTRA=-DWDD_TRACE python -m paper_2212_01309_b200.build --force > /dev/null 2>&1 || exit 1
for c in large live box; do echo "== $c"; python tools/trace_proj.py $c 4096 2>&1 | tail -10; done
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
