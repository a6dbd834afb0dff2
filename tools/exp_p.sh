#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --steps 200 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"
WDD_NVCC_EXTRA=-DWDD_TRACE WDD_LIB_OUT=/tmp/libwdd_trace.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || exit 1
for mf in 32 16 64; do echo "MF=$mf"; WDD_PROJ_MIN_FRAMES=$mf WDD_LIB=/tmp/libwdd_trace.so python tools/trace_ctas.py medium 512; done
WDD_LIB=/tmp/libwdd_trace.so python tools/trace_ctas.py medium 16384
