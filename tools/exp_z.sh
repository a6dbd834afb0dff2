#!/bin/bash
WDD_NVCC_EXTRA="-DWDD_TRACE" WDD_LIB_OUT=/tmp/libwdd_trace.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || exit 1
WDD_LIB=/tmp/libwdd_trace.so python tools/trace_ctas.py large 8192
WDD_LIB=/tmp/libwdd_trace.so python tools/trace_proj.py large 8192 | tail -12
