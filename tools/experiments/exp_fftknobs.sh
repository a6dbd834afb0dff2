python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fk.json 2>/dev/null;
  python -c "
import json,sys;d=json.load(open('gpurun_out/fk.json')); k=d['kernels_isolated']
print(sys.argv[1:], '%.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'rowfft %.3f'%k['rowdft']['ms_per_launch'], 'colfft %.3f'%k['flush']['ms_per_launch'], 'readout %.0f'%d['latency']['readout_us']['p50'])" "$@"; }
run X=0
run WDD_ROWFFT=3,128
run WDD_ROWFFT=2,256
run WDD_ROWFFT=2,128
run WDD_COLFFT=3,128
run WDD_COLFFT=2,256
run WDD_COLFFT=2,128
run WDD_COLFFT_TPC=1
run WDD_COLFFT_TPC=4
run WDD_COLFFT_PF=0
