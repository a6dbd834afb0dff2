python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 300 python bench.py --config medium --steps 400 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mf.json 2>/dev/null;
  python -c "
import json,sys;d=json.load(open('gpurun_out/mf.json'))
print(sys.argv[1:], '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'proj %.3f'%d['roofline']['frac'], 'step %.3f'%d['step_roofline']['frac'], d['clocks']['sm_mhz'])" "$@"; }
run X=0
run WDD_PROJ_MIN_FRAMES=4
run WDD_PROJ_MIN_FRAMES=8
run WDD_PROJ_MIN_FRAMES=12
run WDD_PROJ_MIN_FRAMES=16
run WDD_PROJ_MIN_FRAMES=24
run WDD_PROJ_MIN_FRAMES=32
run X=0
