# per-CTA timelines (trace build) of lone batches (default and latency grids) and of the Medium chain
WDD_NVCC_EXTRA=-DWDD_TRACE WDD_LIB_OUT=/tmp/libwdd_trace.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || echo BUILD FAIL
for sp in 0 1; do for a in "medium 512 512" "live 1024 1024"; do
  echo "TRACE_SPREAD=$sp"; TRACE_SPREAD=$sp WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_ctas.py $a 2>&1 | tail -7
done; done
