python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
WDD_R_CHUNK_MB=56 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "full_scan or fullsize and large or cadence or spectrum_full" > gpurun_out/ch_pytest.log 2>&1; echo "pytest(chunked) rc=$?"; tail -2 gpurun_out/ch_pytest.log
for c in large box medium; do for mb in 0 32 56 110; do
  WDD_R_CHUNK_MB=$mb timeout 300 python bench.py --config $c --steps 40 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ch.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ch.json'));k=d['kernels_isolated']
print('$c mb=$mb', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'flush %.3f x%d'%(k['flush']['ms_total'], k['flush']['launches']), 'rowfft %.3f'%k['rowdft']['ms_total'], 'readout %.0f'%d['latency']['readout_us']['p50'])"
done; done
