python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in large medium box; do
  timeout 300 python bench.py --config $c --steps 40 --no-cpu-baseline --e2e-steps 1 > gpurun_out/lb.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/lb.json'))
print('$c', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'proj %.3f'%d['roofline']['frac'])"
done
WDD_LIB_OUT=/tmp/libwdd_trace.so WDD_NVCC_EXTRA=-DWDD_TRACE python -c "from paper_2212_01309_b200 import build; build.build(force=True)" > /dev/null 2>&1
WDD_LIB=/tmp/libwdd_trace.so timeout 300 python tools/trace_ctas.py large 65536 65536
