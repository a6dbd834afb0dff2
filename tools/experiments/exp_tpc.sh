# y-FFT k-tiles per CTA with the half plane (WDD_COLFFT_TPC=1 vs the default choice)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for c in box large medium; do for v in 0 1 0 1; do
  st=$([ $c = medium ] && echo 300 || ([ $c = box ] && echo 20 || echo 40))
  WDD_COLFFT_TPC=$v timeout 400 python bench.py --config $c --steps $st --no-cpu-baseline --e2e-steps 1 > gpurun_out/t.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/t.json'))
print('$c tpc=$v', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'rd', d['latency']['readout_us']['p50'], d['kernels_ms'] if 'kernels_ms' in d else '')"
done; done
