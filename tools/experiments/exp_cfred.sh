# y-FFT output stage: transposed-butterfly readout reduction (default build) and more rows per
# load round (WDD_CF_U_NOG): parity / bit-identity tests, then bench lines and kernel times
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAIL
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "knob or full_scan or fullsize or half or spectrum or cadence or overlap" > gpurun_out/cf_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/cf_pytest.log
WDD_NVCC_EXTRA=-DWDD_CF_U_NOG=16 WDD_LIB_OUT=/tmp/libwdd_u16.so python -m paper_2212_01309_b200.build > /dev/null 2>&1 || echo BUILD16 FAIL
run() { lib=$1; shift; c=$1; shift; env WDD_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cf.json 2>/dev/null;
  python -c "
import json;d=json.load(open('gpurun_out/cf.json'));k=d['kernels_isolated']
print('$c', '$lib'.split('/')[-1], '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'], 'rowfft %.3f'%k['rowdft']['ms_per_launch'], 'colfft %.3f'%k['flush']['ms_per_launch'], 'readout %.0f'%d['latency']['readout_us']['p50'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
D=paper_2212_01309_b200/_lib/libwdd.so
for c in box large medium; do run $D $c; run /tmp/libwdd_u16.so $c; run $D $c; done
