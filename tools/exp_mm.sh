#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bank or full_scan" 2>&1 | tail -3
timeout 300 python tools/plan_time.py
echo "--- host bank (previous build)"
WDD_LIB=tools/libwdd_hostbank.so timeout 600 python tools/plan_time.py
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
