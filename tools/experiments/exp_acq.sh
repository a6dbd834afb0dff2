python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for A in 1 2 4; do timeout 300 python bench.py --acq-per-graph $A --steps 20 --no-cpu-baseline --e2e-steps 1 > gpurun_out/acq_$A.json 2>/dev/null; done
timeout 300 python bench.py --config large --steps 40 --no-cpu-baseline --e2e-steps 1 > gpurun_out/acq_large.json 2>/dev/null
timeout 300 python bench.py --config live --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/acq_live.json 2>/dev/null
for f in acq_1 acq_2 acq_4 acq_large acq_live; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'))
print('$f', '%.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'step frac %.3f'%d['step_roofline']['frac'], 'proj frac %.3f'%d['roofline']['frac'], 'share %.3f'%d['roofline']['share_of_step'], 'readout', d['latency']['readout_us'], {n:(round(v['ms_per_launch'],4) if v['ms_per_launch'] else None) for n,v in d['kernels_isolated'].items()}, d['clocks']['sm_mhz'])"; done
