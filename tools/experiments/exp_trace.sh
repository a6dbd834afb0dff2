python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_shards.py -q -p no:cacheprovider -k "one_rank_comm" 2>&1 | tail -3
WDD_LIB_OUT=/tmp/libwdd_trace.so WDD_NVCC_EXTRA=-DWDD_TRACE python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > /dev/null 2>&1; echo build $?
for c in large medium box; do echo "== $c"; WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_proj.py $c 8192 200 2>&1 | tail -12; done
