# Medium readout-tail knobs (bench.py --config medium, 300 steps each)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 300 python bench.py --config medium --steps 300 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mk.json 2>/dev/null;
  python -c "
import json,sys;d=json.load(open('gpurun_out/mk.json')); k=d['kernels_isolated']
print(sys.argv[1:], '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'rowfft %.1f'%(1e3*k['rowdft']['ms_per_launch']), 'flush %.1f'%(1e3*k['flush']['ms_per_launch']), 'img %.1f'%(1e3*k['finalize']['ms_per_launch']))" "$@"; }
run X=0
run WDD_IMG=unfused
run WDD_IMG_CS=8
run WDD_IMG_NT=256
run WDD_ROWFFT=3,128
run WDD_ROWFFT=4,256
run WDD_COLFFT=4,256
run WDD_COLFFT_TPC=2
run WDD_ROWFFT_PDL=1
run X=1
