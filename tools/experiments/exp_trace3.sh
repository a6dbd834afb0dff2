WDD_LIB_OUT=/tmp/libwdd_trace.so WDD_NVCC_EXTRA=-DWDD_TRACE python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > /dev/null 2>&1; echo build $?
for c in large medium; do WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_proj.py $c 8192 0 > gpurun_out/trace3_$c.txt 2>&1; done
wc -l gpurun_out/trace3_*.txt
