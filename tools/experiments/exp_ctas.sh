WDD_LIB_OUT=/tmp/libwdd_trace.so WDD_NVCC_EXTRA=-DWDD_TRACE python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > /dev/null 2>&1; echo build $?
WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_ctas.py large 65536 65536
WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_ctas.py box 8192 16384
WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_ctas.py medium 512 16384
