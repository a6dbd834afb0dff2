# per-CTA timelines (trace build) of lone batches and of the Medium chain
WDD_NVCC_EXTRA=-DWDD_TRACE WDD_LIB_OUT=/tmp/libwdd_trace.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || echo BUILD FAIL
for a in "medium 512 512" "medium 512 16384" "live 1024 1024" "box 8192 8192"; do
  WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_ctas.py $a 2>&1 | tail -6
done
