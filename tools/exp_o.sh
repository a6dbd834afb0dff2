#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
WDD_NVCC_EXTRA=-DWDD_TRACE WDD_LIB_OUT=/tmp/libwdd_trace.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || exit 1
for b in 512 16384; do WDD_LIB=/tmp/libwdd_trace.so python tools/trace_ctas.py medium $b; done
WDD_PROJ_MIN_FRAMES=8 WDD_LIB=/tmp/libwdd_trace.so python tools/trace_ctas.py medium 512
